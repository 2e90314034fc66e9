cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
PMGR_TEST_LOGDIR=gpurun_out timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -s > gpurun_out/t_multiproc.log 2>&1; echo "multiproc rc=$?"
tail -5 gpurun_out/t_multiproc.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "setup_bitwise or option_variants or laplacian or production_parity or dist" > gpurun_out/t_setup.log 2>&1; echo "setup tests rc=$?"
tail -3 gpurun_out/t_setup.log
PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 > gpurun_out/setup_trace_c4b.txt 2>&1
grep "=== setup" gpurun_out/setup_trace_c4b.txt
export PMGR_NO_GRAPHS=1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_arnoldi --launch-skip 138 -c 1 --csv python bench.py --ncu --warmup 0 > gpurun_out/ncu_arnoldi_j138.csv 2> gpurun_out/ncu_arnoldi_j138.err; echo "ncu rc=$?"
grep -E "dram__|gpu__time" gpurun_out/ncu_arnoldi_j138.csv | tail -5
