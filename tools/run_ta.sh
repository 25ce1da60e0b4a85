mkdir -p gpurun_out
python -m pytest tests/test_gpu_filter_tc.py -x -q > gpurun_out/ta_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ta_tests.log
L1F_TC_PROF=1 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof5.json 2> gpurun_out/prof5.err
python bench.py --config 5 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b5.json 2> gpurun_out/b5.err
L1F_TC_PROF=1 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof3.json 2> gpurun_out/prof3.err
python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/b3.json 2> gpurun_out/b3.err
