for v in "PMGR_SJ_U=0" "PMGR_SJ_U=4" "PMGR_SJ_U=16" "PMGR_SJ_MIN_ROWS=100000"; do
  env $v python bench.py --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_sj_$v.json 2> gpurun_out/bench_sj_$v.err
  echo "== $v rc=$?"
  python - "gpurun_out/bench_sj_$v.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'its', d['gmres_iterations'], 'setup', d['setup_s'], 'conv', d['converged'], d['true_relative_residual'])
for k,v in d['kernels'].items(): print(' ', k, round(v['avg_us'],1), round(v['gbs'],1))
PY
done
v=SJ
PMGR_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --launch-skip 2000 -c 1000 --csv \
  --log-file gpurun_out/launches_$v.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu_$v.log 2>&1
echo "ncu rc=$?"
