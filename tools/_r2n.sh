for c in C2 C3 C5; do
  for v in "PMGR_NO_SJ=1" "PMGR_SJ=1"; do
  env $v python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $v', round(d['value'],3), 'MDOF/s', round(d['ms_per_step'],2), 'ms its', d['gmres_iterations'], d['converged'], 'setup', round(d['setup_s'],3), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
  done
done
