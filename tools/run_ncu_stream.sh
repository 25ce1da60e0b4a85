#!/bin/bash
# cfg3 bench line, then the ncu launch list of the same command and one full capture of the
# streamed reconstruction kernel (each after the plain run exited 0)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err || { echo bench failed; tail gpurun_out/bench_cfg3.err; exit 1; }
python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg3.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['gpu_launches'], d['clocks'], d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recon_stream_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_recon_stream python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
