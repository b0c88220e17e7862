mkdir -p gpurun_out/r2s2
timeout 900 python -m pytest tests/test_warnings.py -q -x > gpurun_out/r2s2/warn.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2s2/gpu_tests.log 2>&1
echo done
