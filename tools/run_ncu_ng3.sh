mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:adm_tc_kernel --launch-skip 2 -c 1 -f -o gpurun_out/r1_cfg3_filter_ng3 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ng3.log 2>&1
