mkdir -p gpurun_out/r2n2b
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2n2b/bench_n2.json 2> gpurun_out/r2n2b/bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tools/peer_check.py > gpurun_out/r2n2b/peer2.json 2> gpurun_out/r2n2b/peer2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29523 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2n2b/bench_ref_n2.json 2> gpurun_out/r2n2b/bench_ref_n2.err
timeout 600 python -m pytest tests/test_gpu_shards.py -q > gpurun_out/r2n2b/shards.log 2>&1
echo done
