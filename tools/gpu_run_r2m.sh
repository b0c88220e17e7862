mkdir -p gpurun_out/r2m
timeout 120 ./tools/bench_greedy > gpurun_out/r2m/bench_greedy.json 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2m/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 2 --family dense > gpurun_out/r2m/probe_dense.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --order 1 > gpurun_out/r2m/probe_desc.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2m/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2m/bench.json 2> gpurun_out/r2m/bench.err
echo done
