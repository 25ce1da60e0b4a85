mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_tests.log
python bench.py > gpurun_out/full_b3.json 2> gpurun_out/full_b3.err
python bench.py --config 5 --no-cpu-baseline > gpurun_out/full_b5.json 2> gpurun_out/full_b5.err
python bench.py --config 4 --no-cpu-baseline > gpurun_out/full_b4.json 2> gpurun_out/full_b4.err
