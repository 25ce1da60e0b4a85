#!/bin/bash
# Round-2 ncu captures (one GPU): launch list of the default bench step, full sets of the cfg3/cfg5
# filter and reconstruction kernels and of the generator.  Each command ran clean without ncu first.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
$B > gpurun_out/r2_pre.json 2> gpurun_out/r2_pre.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg3.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:adm_tc_kernel -s 2 -c 1 -f -o gpurun_out/r2_cfg3_filter $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:generate_kernel -s 1 -c 1 -f -o gpurun_out/r2_cfg3_generate $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:recon_tc_kernel -s 1 -c 1 -f -o gpurun_out/r2_cfg3_recon $B > /dev/null 2>&1
B5="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
ncu --set full --clock-control none --import-source on -k regex:adm_tc_kernel -s 2 -c 1 -f -o gpurun_out/r2_cfg5_filter $B5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:recon_tc_kernel -s 1 -c 1 -f -o gpurun_out/r2_cfg5_recon $B5 > /dev/null 2>&1
ls -la gpurun_out/r2_*
