# C4 launch list (first ~7 GMRES iterations) and full ncu captures of the outer SpMV and the level-1 CSR sweep
export PMGR_NO_GRAPHS=1
T=${1:-c4}
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 700 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --config C4 --ncu --warmup 1 > gpurun_out/${T}_ncu.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bsr3 --launch-skip 0 --launch-count 3 \
    -f -o gpurun_out/${T}_bsr3 python bench.py --config C4 --ncu --warmup 1 > gpurun_out/${T}_ncu2.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_spmv --launch-skip 0 --launch-count 4 \
    -f -o gpurun_out/${T}_spmv python bench.py --config C4 --ncu --warmup 1 > gpurun_out/${T}_ncu3.log 2>&1
