for v in "PMGR_DBUF_CACHE=0" "PMGR_DBUF_CACHE=1" "PMGR_DBUF_CACHE=0" "PMGR_DBUF_CACHE=1"; do
env $v python bench.py --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['gmres_iterations'], 'setup', d['setup_s'], d['clocks']['sm_mhz'], {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done
