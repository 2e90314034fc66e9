cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
timeout 1200 python -m pytest tests -m gpu -x -q -s -k "tma_block or production or multiproc or test_mgr_apply_and_gmres or full_size" --durations=15 > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
grep -E "^\[|passed|failed|rc=|Error|assert" gpurun_out/gputest.log | tail -40
python bench.py --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_c4_tma.json 2> gpurun_out/bench_c4_tma.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_tma.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'its', d['gmres_iterations'], 'setup', d['setup_s'])
for k,v in d['kernels'].items(): print(k, v['avg_us'], v['gbs'])
"
PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 > gpurun_out/setup_trace_c4.txt 2>&1
tail -5 gpurun_out/setup_trace_c4.txt
