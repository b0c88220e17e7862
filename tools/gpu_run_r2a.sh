set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" --durations=15 > gpurun_out/r2a/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
timeout 300 python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2a/probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"intra_fused|token_keys" -c 2 -o gpurun_out/r2a/sp -f python bench.py --steps 1 --warmup 0 --no-extras > gpurun_out/r2a/ncu_sp.log 2>&1
echo done
