mkdir -p gpurun_out/r2z
timeout 300 python tools/probe_intra.py --batches 1024 --check 4 > gpurun_out/r2z/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 4 --family dense > gpurun_out/r2z/probe_dense.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --order 1 > gpurun_out/r2z/probe_desc.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2z/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2z/bench.json 2> gpurun_out/r2z/bench.err
echo done
