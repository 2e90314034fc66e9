timeout 600 python tools/conv_probe2.py C4 32 jac ilu16 r200 fs2 ilu16+r200 ilu16+fs2 tc2 > gpurun_out/p2_c4_32.log 2>&1
timeout 900 python tools/conv_probe2.py C4 64 jac ilu16 r200 ilu16+r200 ilu16+fs2 ilu64 > gpurun_out/p2_c4_64.log 2>&1
timeout 900 python tools/conv_probe2.py C3 64 ilu16+r300 ilu16+fs2 ilu16+fs2+r200 ilu64+r300 r400 > gpurun_out/p2_c3_64.log 2>&1
timeout 1200 python tools/conv_probe2.py C4 128 jac ilu16 ilu16+r200 > gpurun_out/p2_c4_128.log 2>&1
grep -h -v "F rows" gpurun_out/p2_*.log | cut -c1-300
