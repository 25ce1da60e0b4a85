mkdir -p gpurun_out
python -m pytest tests/test_gpu_filter_tc.py -x -q > gpurun_out/ng3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ng3_tests.log
L1F_TC_PROF=1 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ng3_prof3.json 2> gpurun_out/ng3_prof3.err
python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/ng3_b3.json 2> gpurun_out/ng3_b3.err
L1F_TC_NG=2 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/ng2_b3.json 2> gpurun_out/ng2_b3.err
python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/ng3_b2.json 2> gpurun_out/ng3_b2.err
L1F_TC_NG=2 python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/ng2_b2.json 2> gpurun_out/ng2_b2.err
