# quick GPU check of the current tree: gpu tests, C2 bench, optional C4 bench
# usage (under gpurun): bash tools/perf_check.sh TAG [C4]
TAG=${1:-pc}
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/${TAG}_tests.txt
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err
if [ "$2" != "" ]; then
  python bench.py --config $2 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/${TAG}_$2.json 2> gpurun_out/${TAG}_$2.err
fi
python tools/summ.py gpurun_out/${TAG}_*.json
cat gpurun_out/${TAG}_tests.txt
