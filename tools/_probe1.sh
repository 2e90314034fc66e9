set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in "C4 32" "C3 32"; do timeout 900 python tools/conv_probe2.py $c jac gs32 fs2 gal ilu4096 tc2 r300 gs32+fs2 gal+gs32 ; done > gpurun_out/probe_small.log 2>&1
timeout 900 python tools/conv_probe2.py C4 64 jac gs32 fs2 gal ilu16384 r300 gal+gs32 > gpurun_out/probe_c4_64.log 2>&1
timeout 900 python tools/conv_probe2.py C3 64 jac gs32 gal gal+gs32 fs2 ilu16384 > gpurun_out/probe_c3_64.log 2>&1
tail -50 gpurun_out/probe_*.log
