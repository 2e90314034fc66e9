cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 3000 --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_summary.txt 2>&1; head -40 gpurun_out/launches_c4_summary.txt
