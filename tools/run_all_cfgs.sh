mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in 1 2 3 4; do python bench.py --config $c > gpurun_out/all_b$c.json 2> gpurun_out/all_b$c.err; done
python bench.py --config 5 --no-cpu-baseline > gpurun_out/all_b5.json 2> gpurun_out/all_b5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/all_ref3.json 2> gpurun_out/all_ref3.err
