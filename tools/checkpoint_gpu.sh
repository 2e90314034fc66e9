# Official bench lines + profiles for the current tree (run under gpurun).
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/ck_tests.txt
python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/ck_ref.json 2> gpurun_out/ck_ref.err
export PMGR_NO_GRAPHS=1
python bench.py --ncu --warmup 1 > /dev/null 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/ck_launches.csv python bench.py --ncu --warmup 1 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_arnoldi \
    --launch-skip 45 --launch-count 2 -f -o gpurun_out/ck_k_arnoldi python bench.py --ncu --warmup 1 > /dev/null 2>&1
ls -la gpurun_out/
