# C2 bench under several env settings (under gpurun): bash tools/envsweep.sh TAG "A=1 B=2" "A=0" ...
TAG=$1; shift
i=0
for E in "$@"; do
  env $E python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_$i.json 2> gpurun_out/${TAG}_$i.err
  echo "$i: $E"; python tools/summ.py gpurun_out/${TAG}_$i.json 2>/dev/null | head -1
  i=$((i+1))
done
