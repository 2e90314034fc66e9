# full GPU suite + driver-style bench on the current tree
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputest_full.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_full.log
tail -25 gpurun_out/gputest_full.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_c4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'its', d['gmres_iterations'], 'setup', d['setup_s'], 'e2e', d['e2e']['value'])
for k,v in d['kernels'].items(): print(k, v['avg_us'], v['gbs'])
print(d['roofline'])
print(d['cpu_baseline'])
PY
