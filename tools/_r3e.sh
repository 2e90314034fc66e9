python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
PMGR_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --launch-skip 2000 -c 700 --csv \
  --log-file gpurun_out/r02_launches_c4.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_c4.csv > gpurun_out/r02_launches_c4_summary.txt 2>&1
python tools/iter_breakdown.py gpurun_out/r02_launches_c4.csv > gpurun_out/r02_iteration_c4.txt 2>&1
PMGR_NO_GRAPHS=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k_arnoldi --launch-skip 138 -c 1 --csv \
  --log-file gpurun_out/r02_ncu_arnoldi_j138.csv python bench.py --ncu --warmup 0 > gpurun_out/ncu_arn.log 2>&1; echo "arnoldi rc=$?"
grep -v "^==" gpurun_out/r02_ncu_arnoldi_j138.csv | tail -4
for c in C2 C3 C5; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; echo "$c rc=$?"
done
