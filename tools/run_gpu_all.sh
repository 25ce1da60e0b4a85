#!/bin/bash
# all GPU tests, the streamed-path diagnostics and the default bench line (1 GPU)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 600 python tools/diag_streamed.py 3 > gpurun_out/diag3.log 2>&1; tail -9 gpurun_out/diag3.log
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg3.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline_reconstruct']['frac'], json.dumps(d['phases_ms']), d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
