#!/bin/bash
# streamed row filter + reconstruction: parity tests, then the cfg3 bench line (1 GPU)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_streamed.py -x -q > gpurun_out/streamed_tests.log 2>&1
echo "tests rc=$?"
tail -15 gpurun_out/streamed_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_streamed.json 2> gpurun_out/bench_streamed.err
echo "bench rc=$?"
tail -3 gpurun_out/bench_streamed.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_streamed.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], json.dumps(d["phases_ms"]), d["roofline"]["frac"], d["roofline_reconstruct"]["frac"])
PY
