#!/bin/bash
# the N-GPU driver at world 1 (plain and forced sharded), then the ncu launch list of the
# default bench command restricted to the library's kernels (after the plain run exited 0)
mkdir -p gpurun_out
bash tools/run_dist1.sh
for f in dist1 dist1s dist1r; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d.get('value'), d.get('ms_per_step'), d.get('config',{}).get('parallelism'), (d.get('e2e') or {}).get('value'), d.get('gpu_launches'), (d.get('roofline') or {}).get('frac'))" || tail -5 gpurun_out/$f.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:adm_tc|recon_|unit_scale|gather|split_|strip_p0|build_factors|sum_items|gate' -c 60 --csv \
  --log-file gpurun_out/launches_cfg3_v5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
