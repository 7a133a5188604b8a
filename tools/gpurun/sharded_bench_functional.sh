# gpurun recipe: the sharded bench code path on ONE GPU (functional check, not a measurement):
# two ranks on GPU 0 over gloo, peer mode (CUDA IPC, host barriers) and NCCL-free exchange-less path
BENCH_FUNCTIONAL_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --config c4 --qubits 13 --steps 1 --warmup 1 --no-cpu > gpurun_out/shard_func.json 2> gpurun_out/shard_func.err
echo "rc=$?" >> gpurun_out/shard_func.err
