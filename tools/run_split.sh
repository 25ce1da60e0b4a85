set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_filter_tc.py -x -q > gpurun_out/split_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/split_tests.log
L1F_TC_PROF=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/split_prof.json 2> gpurun_out/split_prof.err
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/split_b3.json 2> gpurun_out/split_b3.err
python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/split_b5.json 2> gpurun_out/split_b5.err
