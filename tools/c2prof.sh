# C2 full ncu captures of the level-0 block sweeps, the outer SpMV, the
# level-1 CSR sweep and the dense collapsed matvec (under gpurun)
export PMGR_NO_GRAPHS=1
T=${1:-c2}
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bsr3 --launch-skip 30 --launch-count 3 \
    -f -o gpurun_out/${T}_bsr3 python bench.py --ncu --warmup 1 > gpurun_out/${T}_ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_spmv<32" --launch-skip 20 --launch-count 2 \
    -f -o gpurun_out/${T}_spmv32 python bench.py --ncu --warmup 1 > gpurun_out/${T}_ncu2.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_dense --launch-skip 20 --launch-count 2 \
    -f -o gpurun_out/${T}_dense python bench.py --ncu --warmup 1 > gpurun_out/${T}_ncu3.log 2>&1
ls -la gpurun_out/
