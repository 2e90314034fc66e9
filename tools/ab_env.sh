# A/B of one env knob on the C2 bench (under gpurun), values round-robin twice:
#   bash tools/ab_env.sh TAG VAR V1 V2 [V3 ...]
TAG=$1; VAR=$2; shift 2
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/${TAG}_tests.txt
for R in 1 2; do
  for V in "$@"; do
    env $VAR=$V python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_${V}_${R}.json 2> gpurun_out/${TAG}_${V}_${R}.err
  done
done
python tools/summ.py gpurun_out/${TAG}_*.json
cat gpurun_out/${TAG}_tests.txt
