timeout 1500 python tools/conv_probe2.py C4 128 r200 r300 fs2 tc2 r200+tc2 r200+fs2 r300+tc2 > gpurun_out/p3_c4_128.log 2>&1
timeout 900 python tools/conv_probe2.py C3 64 ilu16+fs2+r300 ilu16+fs2+tc2+r200 ilu16+tc2+r200 ilu8+fs2+r200 ilu32+fs2+r200 > gpurun_out/p3_c3_64.log 2>&1
timeout 900 python tools/conv_probe2.py C5 128 jac r200 r200+tc2 > gpurun_out/p3_c5_128.log 2>&1
grep -h -v "F rows" gpurun_out/p3_*.log | cut -c1-250
