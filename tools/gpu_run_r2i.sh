mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2i/gpu_tests.log 2>&1
timeout 600 python tools/probe_c5.py --batches 64 --check 0 --inter-batches 8 > gpurun_out/r2i/c5.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2i/bench.json 2> gpurun_out/r2i/bench.err
echo done
