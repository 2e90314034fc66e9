# C4 bench line for profiles/ (under gpurun)
python bench.py --config C4 --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/ck_c4.json 2> gpurun_out/ck_c4.err
