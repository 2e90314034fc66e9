export PMGR_NO_GRAPHS=1
mkdir -p /tmp/reps
run() { # tag, kernel regex, skip
  tag=$1; k=$2; skip=$3
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled -k "$k" --launch-skip $skip -c 1 \
     -o /tmp/reps/c4_$tag -f python bench.py --ncu --warmup 0 > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page details > gpurun_out/r02_ncu_c4_${tag}_details.txt 2>&1
  ncu -i /tmp/reps/c4_$tag.ncu-rep --page source --csv > gpurun_out/r02_ncu_c4_${tag}_source.csv 2>&1
}
run sjs_l1 'regex:k_sjs<\(int\)8, .*OpResidual' 0
run sj_blk 'regex:k_sj<\(int\)2, \(int\)2, .*OpJacobi>' 1
run sj_outer 'regex:k_sj<\(int\)8, \(int\)2, .*OpY' 1
du -sh gpurun_out
