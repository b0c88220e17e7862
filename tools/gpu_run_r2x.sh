mkdir -p gpurun_out/r2x
timeout 300 python tools/probe_intra.py --batches 1024 --check 4 --order 1 > gpurun_out/r2x/probe_desc.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2x/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --family dense > gpurun_out/r2x/probe_dense.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2x/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2x/bench.json 2> gpurun_out/r2x/bench.err
echo done
