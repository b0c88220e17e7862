mkdir -p gpurun_out/r2i2
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2i2/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 2 --family dense > gpurun_out/r2i2/probe_dense.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 4 --order 1 > gpurun_out/r2i2/probe_desc.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2i2/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2i2/bench.json 2> gpurun_out/r2i2/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2i2/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
echo done
