# launch list (one iteration's kernels) with the sliced jagged copy at default thresholds, and without
for v in "PMGR_SJ_UB=2" "PMGR_NO_SJ=1"; do
env $v PMGR_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --launch-skip 2000 -c 1400 --csv \
  --log-file gpurun_out/launches_$v.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu_$v.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_$v.csv > gpurun_out/launches_${v}_summary.txt 2>&1; head -45 gpurun_out/launches_${v}_summary.txt
done
PMGR_HIER_STATS=1 PMGR_SJ_UB=2 python bench.py --no-cpu-baseline --steps 1 --warmup 1 2>&1 | grep "pmgr\]" | head -60
