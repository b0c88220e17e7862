mkdir -p gpurun_out/r2v
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2v/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2v/bench.json 2> gpurun_out/r2v/bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --samples 4194304 > gpurun_out/r2v/bench_4m.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r2v/launches_4m.csv python bench.py --steps 1 --warmup 3 --no-extras --samples 4194304 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r2v/launches.csv python bench.py --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
echo done
