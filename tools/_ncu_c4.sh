cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
export PMGR_NO_GRAPHS=1
for spec in "bsr3p:regex:k_bsr3p<OpJacobi," "csr32:regex:k_spmv<32, 0, OpResidual, int" "outer:regex:k_bsr3<OpResidual" "arnoldi:regex:k_arnoldi"; do
  tag=${spec%%:*}; k=${spec#*:}
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k "$k" -c 1 \
     -o gpurun_out/c4_$tag -f python bench.py --ncu --warmup 0 > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
done
ls -la gpurun_out/*.ncu-rep
