mkdir -p gpurun_out/n2c
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/peer_check.py > gpurun_out/n2c/peer2.json 2> gpurun_out/n2c/peer2.err
echo done
