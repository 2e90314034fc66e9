cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
for e in "X=1" "PMGR_DIST_REPLICATE_ROWS=300" "PMGR_COLLAPSE_ROWS=300" "PMGR_COLLAPSE_ROWS=300 PMGR_DIST_REPLICATE_ROWS=300" "PMGR_DIST_REPLICATE_ROWS=100000"; do
  echo "== $e"; env $e python tools/_dbg_dist.py 2>&1 | grep -v "F rows"
done
timeout 1500 python -m pytest tests -m gpu -q -x -k "setup_bitwise or option_variants or laplacian or production_parity" > gpurun_out/t_setup2.log 2>&1; echo "setup tests rc=$?"
tail -3 gpurun_out/t_setup2.log
SETUP_REPS=3 PMGR_SETUP_TRACE=1 python tools/setup_trace.py C4 2>&1 | grep "=== setup\|spgemm"| tail -12
