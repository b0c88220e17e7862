mkdir -p gpurun_out/r2t
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2t/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2t/bench.json 2> gpurun_out/r2t/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r2t/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
echo done
