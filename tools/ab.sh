# A/B of an env knob on C2 and C4 (under gpurun): bash tools/ab.sh TAG VAR VAL_A VAL_B [C4]
TAG=$1; VAR=$2
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/${TAG}_tests.txt
for V in $3 $4; do
  env $VAR=$V python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_${V}_c2.json 2> gpurun_out/${TAG}_${V}_c2.err
  if [ "$5" != "" ]; then env $VAR=$V python bench.py --config $5 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/${TAG}_${V}_$5.json 2> gpurun_out/${TAG}_${V}_$5.err; fi
done
python tools/summ.py gpurun_out/${TAG}_*.json
cat gpurun_out/${TAG}_tests.txt
