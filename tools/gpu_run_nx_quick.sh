N=$1
mkdir -p gpurun_out/q$N
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N tools/peer_check.py > gpurun_out/q$N/peer.json 2> gpurun_out/q$N/peer.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N --steps 10 --warmup 3 --no-extras > gpurun_out/q$N/bench.json 2> gpurun_out/q$N/bench.err
timeout 600 python -m pytest tests/test_gpu_shards.py -q > gpurun_out/q$N/shards.log 2>&1
echo done
