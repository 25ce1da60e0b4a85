mkdir -p gpurun_out
for i in 1 2; do python bench.py --config 5 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b5_$i.json 2> gpurun_out/b5_$i.err; done
L1F_TC_PROF=1 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof5.json 2> gpurun_out/prof5.err
