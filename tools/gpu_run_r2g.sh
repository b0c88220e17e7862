mkdir -p gpurun_out/r2g
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2g/probe.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 2 --family dense > gpurun_out/r2g/probe_dense.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 2 --order 1 > gpurun_out/r2g/probe_desc.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2g/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2g/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:intra_fused -c 1 -o gpurun_out/r2g/k1 python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2g/ncu_k1.log 2>&1
echo done
