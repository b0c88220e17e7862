#!/bin/bash
# K0 instruction-diet variants: parity of the product build, then per-variant
# step time and cost-pass launch times (tools/exp_variants.sh).
mkdir -p gpurun_out/k0
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/k0/gpu_tests.log 2>&1
bash tools/exp_variants.sh cost_stream base lean lean16 base lean lean16 > gpurun_out/k0/variants.log 2>&1
echo done
