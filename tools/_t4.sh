cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
PMGR_TEST_LOGDIR=gpurun_out timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -s > gpurun_out/t_multiproc.log 2>&1; echo "multiproc rc=$?"
tail -5 gpurun_out/t_multiproc.log
SETUP_REPS=1 PMGR_SETUP_TRACE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_launches.csv python tools/setup_trace.py C4 > gpurun_out/setup_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/setup_launches.csv > gpurun_out/setup_launches_summary.txt 2>&1; head -30 gpurun_out/setup_launches_summary.txt
rm -f gpurun_out/setup_launches.csv
