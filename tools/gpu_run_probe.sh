#!/bin/bash
# partition-kernel probe (per-batch stamps: kept-order write-out), parity, bench step
mkdir -p gpurun_out/probe5
timeout 600 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/probe5/mixed.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/probe5/bench.json 2>/dev/null
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/probe5/tests.log 2>&1
echo done
