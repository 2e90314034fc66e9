# C4 A/B of one env knob (under gpurun): bash tools/ab_c4.sh TAG VAR V1 V2 ...
TAG=$1; VAR=$2; shift 2
for V in "$@"; do
  env $VAR=$V python bench.py --config C4 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/${TAG}_${V}_C4.json 2> gpurun_out/${TAG}_${V}_C4.err
done
python tools/summ.py gpurun_out/${TAG}_*_C4.json
