mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pdl/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/pdl/bench.json 2> gpurun_out/pdl/bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/pdl/bench2.json 2> /dev/null
echo done
