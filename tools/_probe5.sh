cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
SETUP_REPS=3 PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 2>&1 | grep "=== setup\|coarsest"
timeout 1500 python tools/conv_probe2.py C4 128 r300+fs3 r500+fs2 r600+fs2 r400+fs3 r500+fs3 r300+fs4 > gpurun_out/p5_c4_128.log 2>&1
grep -h -v "F rows" gpurun_out/p5_c4_128.log | cut -c1-200
