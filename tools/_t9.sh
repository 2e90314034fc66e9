cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/t9.log 2>&1; echo "rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/t9.log | tail -20
PMGR_OVERLAP=0 timeout 600 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/t9b.log 2>&1; echo "no-overlap dist rc=$?"; tail -2 gpurun_out/t9b.log
