cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
PMGR_TEST_LOGDIR=gpurun_out timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_reference_api.py -q -s > gpurun_out/t6.log 2>&1; echo "rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/t6.log | tail -20
SETUP_REPS=3 PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 > gpurun_out/setup_trace_c4c.txt 2>&1
grep "=== setup" gpurun_out/setup_trace_c4c.txt
