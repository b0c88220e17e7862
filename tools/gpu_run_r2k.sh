mkdir -p gpurun_out/r2k
timeout 120 ./tools/bench_greedy > gpurun_out/r2k/bench_greedy.json 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 1 > gpurun_out/r2k/probe.log 2>&1
echo done
