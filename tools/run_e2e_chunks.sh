mkdir -p gpurun_out
for c in 8 16 32; do
  python bench.py --no-cpu-baseline --steps 5 --e2e-chunks $c > gpurun_out/e2e_c$c.json 2> gpurun_out/e2e_c$c.err
done
