python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/rp_tests.txt
for R in 1 2; do
PMGR_LIB=$PWD/build/ab/base.so python bench.py --no-cpu-baseline --steps 5 > gpurun_out/rp_A$R.json 2>/dev/null
PMGR_LIB=$PWD/build/ab/rp.so python bench.py --no-cpu-baseline --steps 5 > gpurun_out/rp_B$R.json 2>/dev/null
PMGR_BSR_RMINB=0 PMGR_LIB=$PWD/build/ab/rp.so python bench.py --no-cpu-baseline --steps 5 > gpurun_out/rp_C$R.json 2>/dev/null
done
python tools/summ.py gpurun_out/rp_*.json
cat gpurun_out/rp_tests.txt
