# round-2 artefacts on the current tree: driver-style bench line, reference arm, launch list, ncu details of the sliced jagged kernels
python bench.py > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
PMGR_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --launch-skip 2000 -c 700 --csv \
  --log-file gpurun_out/r02_launches_c4.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu_launches.log 2>&1; echo "launch list rc=$?"
python tools/launch_summary.py gpurun_out/r02_launches_c4.csv > gpurun_out/r02_launches_c4_summary.txt 2>&1
python tools/iter_breakdown.py gpurun_out/r02_launches_c4.csv > gpurun_out/r02_iteration_c4.txt 2>&1
export PMGR_NO_GRAPHS=1
mkdir -p /tmp/reps
run() { tag=$1; k=$2; skip=$3
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "$k" --launch-skip $skip -c 1 \
     -o /tmp/reps/c4_$tag -f python bench.py --ncu --warmup 0 > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page details > gpurun_out/r02_ncu_c4_${tag}_details.txt 2>&1
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
for k in ('dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct'):
    if k in h: print(k, rows[1][h.index(k)], v[h.index(k)])
" > gpurun_out/r02_ncu_c4_${tag}_dram.txt 2>&1
}
run sj_blocks 'regex:k_sj<\(int\)2, \(int\)2, .*OpJacobi>' 1
run sjs_level1 'regex:k_sjs<\(int\)8, .*OpResidual' 0
run sj_outer 'regex:k_sj<\(int\)8, \(int\)2, .*OpY' 1
cat gpurun_out/r02_ncu_c4_*_dram.txt
