mkdir -p gpurun_out
for i in 1 2; do
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/side0_$i.json 2>/dev/null
L1F_SIDE_GATHER=1 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/side1_$i.json 2>/dev/null
done
