cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
export PMGR_NO_GRAPHS=1
mkdir -p /tmp/reps
for spec in 'csr32:regex:k_spmv<\(int\)32, \(bool\)0, .*OpResidual, int,' 'bsr3t:regex:k_bsr3t<.*OpResidual'; do
  tag=${spec%%:*}; k=${spec#*:}
  PMGR_BSR_TPW=2 PMGR_BSR_STAGES=2 PMGR_BSR_CPS=3 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "$k" -c 1 \
     -o /tmp/reps/c4_$tag -f python bench.py --ncu --warmup 0 > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page details > gpurun_out/ncu_c4_${tag}_details.txt 2>&1
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_c4_${tag}_raw.csv 2>&1
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page source --csv > gpurun_out/ncu_c4_${tag}_source.csv 2>&1
done
du -sh gpurun_out
