mkdir -p gpurun_out/r2f
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2f/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --family dense > gpurun_out/r2f/probe_dense.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2f/gpu_tests.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r2f/launches.csv python tools/probe_intra.py --batches 1024 --check 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r2f/launches_dense.csv python tools/probe_intra.py --batches 1024 --check 0 --family dense > /dev/null 2>&1
echo done
