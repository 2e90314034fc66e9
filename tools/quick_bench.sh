python -m pytest tests -m gpu -x -q 2>&1 | tail -1 > gpurun_out/qt.txt
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/ao.json 2>gpurun_out/ao.err
python - <<PY
import json
d=json.loads(open("gpurun_out/ao.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["e2e"]["ms_per_step"], d["config"]["gmres_iterations"])
for k,v in d["kernels"].items(): print(k, round(v["avg_us"],2), round(v["gbs"] or 0))
PY
cat gpurun_out/qt.txt
