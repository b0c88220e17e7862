# multi-GPU evidence: bench at N GPUs (torchrun, one process per GPU), the
# reference arm at N, and the peer-exchange check
N=$1
mkdir -p gpurun_out/fn$N
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/fn$N/bench.json 2> gpurun_out/fn$N/bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --impl reference --gpus $N --steps 3 --warmup 3 > gpurun_out/fn$N/bench_ref.json 2> gpurun_out/fn$N/bench_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N tools/peer_check.py > gpurun_out/fn$N/peer.json 2> gpurun_out/fn$N/peer.err
timeout 600 python -m pytest tests/test_gpu_shards.py -q > gpurun_out/fn$N/shards.log 2>&1
echo done
