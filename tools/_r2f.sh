sel="test_spmv or test_amg_laplacian_bitwise or test_mgr_apply_and_gmres or test_mgr_option_variants or test_all_c_level or test_empty_and_tiny or test_distributed_apply or test_halo_overlap or test_distributed_gmres or test_apply_is_linear"
for g in 1 4; do
PMGR_SJ_MIN_NNZ=1 PMGR_SJ_MIN_ROWS=1 PMGR_SJ_G=$g timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "$sel" > gpurun_out/sj_forced_g$g.log 2>&1
echo "forced g=$g rc=$?"; tail -3 gpurun_out/sj_forced_g$g.log
done
for v in "PMGR_SJ_G=1" "PMGR_SJ_G_MEAN=64 PMGR_SJ_GBIG=2" "PMGR_SJ_G_MEAN=64 PMGR_SJ_GBIG=4" "PMGR_SJ_G_MEAN=64 PMGR_SJ_GBIG=8" "PMGR_SJ_G_MEAN=64 PMGR_SJ_GBIG=4 PMGR_SJ_U=4"; do
  t=$(echo $v | tr ' =' '__')
  env $v python bench.py --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_sj_$t.json 2> gpurun_out/bench_sj_$t.err
  echo "== $v rc=$?"
  python - "gpurun_out/bench_sj_$t.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'its', d['gmres_iterations'], 'setup', d['setup_s'], 'conv', d['converged'], d['true_relative_residual'])
for k,v in d['kernels'].items(): print(' ', k, round(v['avg_us'],1), round(v['gbs'],1))
PY
  env $v PMGR_NO_GRAPHS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --launch-skip 2000 -c 700 --csv \
    --log-file gpurun_out/launches_$t.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu_$t.log 2>&1
  python tools/iter_breakdown.py gpurun_out/launches_$t.csv | head -14
done
