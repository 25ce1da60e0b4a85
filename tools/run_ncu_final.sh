mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pre.json 2> gpurun_out/ncu_pre.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:adm_tc_kernel --launch-skip 2 -c 1 -f -o gpurun_out/r1_cfg3_filter_ng3_v2 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:recon_tc_kernel --launch-skip 2 -c 1 -f -o gpurun_out/r1_cfg3_recon_v4 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r.log 2>&1
ncu --set full --clock-control none -k regex:gather -c 4 -f -o gpurun_out/r1_cfg3_gather_v1 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_g.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_cfg3_v4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
