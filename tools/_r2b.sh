# SJ format: forced everywhere on the small parity tests, then default thresholds at C4
PMGR_SJ_MIN_NNZ=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "test_spmv or test_amg_laplacian_bitwise or test_mgr_apply_and_gmres or test_mgr_option_variants or test_all_c_level or test_empty_and_tiny or test_distributed_apply or test_halo_overlap or test_distributed_gmres or test_apply_is_linear" > gpurun_out/sj_forced.log 2>&1
echo "forced rc=$?"; tail -15 gpurun_out/sj_forced.log
for v in "PMGR_NO_SJ=1" "PMGR_SJ_UB=3" "PMGR_SJ_UB=2"; do
  env $v python bench.py --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_sj_$v.json 2> gpurun_out/bench_sj_$v.err
  echo "== $v rc=$?"
  python - "gpurun_out/bench_sj_$v.json" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'its', d['gmres_iterations'], 'setup', d['setup_s'], 'conv', d['converged'], d['true_relative_residual'])
for k,v in d['kernels'].items(): print(' ', k, round(v['avg_us'],1), round(v['gbs'],1))
PY
done
