set -x
mkdir -p gpurun_out/r2b
timeout 300 python tools/probe_intra.py --batches 1024 --check 4 > gpurun_out/r2b/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 64 --check 4 --order 1 > gpurun_out/r2b/probe_desc.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" --durations=10 > gpurun_out/r2b/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
echo done
