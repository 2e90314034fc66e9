set -x
python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err
python bench.py --config C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err
export PMGR_NO_GRAPHS=1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 700 --csv --log-file gpurun_out/c4_launches.csv python bench.py --config C4 --ncu --warmup 1 > gpurun_out/c4_ncu.log 2>&1
