cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
SETUP_REPS=4 PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 > gpurun_out/setup_trace_c4d.txt 2>&1
grep "=== setup" gpurun_out/setup_trace_c4d.txt
SETUP_REPS=4 python tools/setup_trace.py C4 2>&1 | grep "=== setup"
PMGR_POOL_KEEP=0 SETUP_REPS=3 python tools/setup_trace.py C4 2>&1 | grep "=== setup"
