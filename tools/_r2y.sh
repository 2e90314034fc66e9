timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_full.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest_full.log
SETUP_REPS=3 PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 2>&1 | grep -E "=== setup" | tail -2
python bench.py --no-cpu-baseline --steps 3 --warmup 2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['gmres_iterations'], 'setup', d['setup_s'], d['clocks']['sm_mhz'], {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
