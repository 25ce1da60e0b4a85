mkdir -p gpurun_out
for i in 1 2; do
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/e2e_ng3_$i.json 2> /dev/null
L1F_TC_NG=2 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/e2e_ng2_$i.json 2> /dev/null
done
