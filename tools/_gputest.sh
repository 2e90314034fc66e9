cd paper_1904_05960_b200/csrc && make -j16 > /dev/null 2>&1; cd ../..
timeout 2400 python -m pytest tests -m gpu -x -q -s --durations=15 > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
tail -n 40 gpurun_out/gputest.log
