# C4 bench under several env settings (under gpurun): bash tools/envsweep4.sh TAG CFG "A=1 B=2" "A=0" ...
TAG=$1; CFG=$2; shift; shift
i=0
for E in "$@"; do
  env $E python bench.py --config $CFG --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/${TAG}_$i.json 2> gpurun_out/${TAG}_$i.err
  echo "$i: $E"; python tools/summ.py gpurun_out/${TAG}_$i.json 2>/dev/null
  i=$((i+1))
done
