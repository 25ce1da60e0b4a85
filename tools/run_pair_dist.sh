mkdir -p gpurun_out
for i in 1 2; do
L1F_FORCE_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2951$i bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/pd_on_$i.json 2> gpurun_out/pd_on_$i.err
L1F_FILTER_PAIR=0 L1F_FORCE_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2952$i bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/pd_off_$i.json 2> gpurun_out/pd_off_$i.err
done
