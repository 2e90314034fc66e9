timeout 1500 python tools/conv_probe2.py C4 128 r300+fs2 r400+fs2 r200+fs3 r300+fs3 > gpurun_out/p4_c4_128.log 2>&1
timeout 900 python tools/conv_probe2.py C3 64 ilu16+fs3+r300 ilu16+fs2+r400 ilu16+fs2+r300+post > gpurun_out/p4_c3_64.log 2>&1
timeout 900 python tools/conv_probe2.py C4 32 r300+fs2 r200+fs2 > gpurun_out/p4_c4_32.log 2>&1
timeout 900 python tools/conv_probe2.py C3 32 ilu16+fs2+r300 > gpurun_out/p4_c3_32.log 2>&1
timeout 900 python tools/conv_probe2.py C5 128 r300 fs2+r200 > gpurun_out/p4_c5_128.log 2>&1
grep -h -v "F rows" gpurun_out/p4_*.log | cut -c1-250
