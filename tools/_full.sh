cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
timeout 2700 python -m pytest tests -m gpu -q -s --durations=25 > gpurun_out/gputest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_full.log
grep -E "^\[|passed|failed|rc=|Error" gpurun_out/gputest_full.log | tail -60
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; echo "ref rc=$?"
tail -c 600 gpurun_out/ref_c4.json
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4_full.json 2> gpurun_out/bench_c4_full.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_c4_full.json
nproc; lscpu | grep "Model name"
