mkdir -p gpurun_out
L1F_TC_PROF=1 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof3.json 2> gpurun_out/prof3.err
