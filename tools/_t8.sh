cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
SETUP_REPS=4 PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 > gpurun_out/setup_trace_c4e.txt 2>&1
grep "=== setup" gpurun_out/setup_trace_c4e.txt
grep "spgemm numeric\|spgemm symbolic\|spgemm sort" gpurun_out/setup_trace_c4e.txt | awk '{print $3, $(NF-1)}' | sort -k2 -n -r | head -12
timeout 900 python -m pytest tests -m gpu -q -x -k "setup_bitwise or production_parity" 2>&1 | tail -2
