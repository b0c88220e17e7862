mkdir -p gpurun_out/r2p2
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2p2/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --family dense > gpurun_out/r2p2/probe_dense.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --order 1 > gpurun_out/r2p2/probe_desc.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2p2/gpu_tests.log 2>&1
echo done
