mkdir -p gpurun_out/r2d
timeout 300 python tools/probe_intra.py --batches 1024 --check 2 > gpurun_out/r2d/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 148 --check 0 > gpurun_out/r2d/probe148.log 2>&1
echo done
