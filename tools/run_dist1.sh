mkdir -p gpurun_out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/dist1.json 2> gpurun_out/dist1.err
L1F_FORCE_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/dist1s.json 2> gpurun_out/dist1s.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/dist1r.json 2> gpurun_out/dist1r.err
