mkdir -p gpurun_out
python -m pytest tests/test_gpu_filter_pair.py tests/test_gpu_pipeline.py tests/test_gpu_host_pipeline.py -x -q > gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
for c in 2 3; do python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/pair_b$c.json 2>/dev/null; done
L1F_FORCE_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/pair_dist1s.json 2> gpurun_out/pair_dist1s.err
