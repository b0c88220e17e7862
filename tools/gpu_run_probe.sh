#!/bin/bash
# partition-kernel probe (per-batch stamps), parity, bench step
mkdir -p gpurun_out/probe4
timeout 600 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/probe4/mixed.log 2>&1
timeout 600 python tools/probe_intra.py --batches 1024 --check 3 --family dense > gpurun_out/probe4/dense.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/probe4/tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/probe4/bench.json 2>/dev/null
DTB_LIB_PATH=$PWD/build/obj_DTB_DEBUG_CHECKS/libdisttrain_b200.so timeout 900 python -m pytest tests -q -m gpu -x -k "dense or kept or fullsize" > gpurun_out/probe4/tests_debug.log 2>&1
echo done
