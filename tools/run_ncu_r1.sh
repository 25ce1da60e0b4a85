# one ncu --set full capture per top kernel (cfg3 filter, cfg3 recon, cfg5 recon) + the cfg3 launch list
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pre.json 2> gpurun_out/ncu_pre.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:adm_tc_kernel --launch-skip 2 -c 1 -f -o gpurun_out/r1_cfg3_filter_v3 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:recon_tc_kernel --launch-skip 2 -c 1 -f -o gpurun_out/r1_cfg3_recon_v3 \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_cfg3_v3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:recon_tc_kernel -c 1 -f -o gpurun_out/r1_recon_k200_v1 \
  python tools/time_recon.py 32768 32768 200 > gpurun_out/ncu_r5.log 2>&1
