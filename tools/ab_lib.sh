# A/B(/C...) of builds of libpmgr.so on the same box (under gpurun):
#   bash tools/ab_lib.sh TAG LIB_A LIB_B [LIB_C ...]
# runs the libraries round-robin twice so box drift shows up; prints
# ms/step and the instrumented kernel times (tools/summ.py).
TAG=$1; shift
for R in 1 2; do
  i=0
  for LIB in "$@"; do
    L=$(printf "\\x$(printf %x $((65 + i)))"); i=$((i + 1))
    PMGR_LIB=$PWD/$LIB python bench.py --no-cpu-baseline --steps 5 > gpurun_out/${TAG}_${L}${R}.json 2> gpurun_out/${TAG}_${L}${R}.err
  done
done
python tools/summ.py gpurun_out/${TAG}_*.json
