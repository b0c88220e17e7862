#!/bin/bash
# Cost-pass prefix scan: one 16-byte word per lane and step (DTB_COST_SCAN_L=4,
# conflict-free) vs two (L=8, lanes 32 B apart: 2-way bank conflicts).
mkdir -p gpurun_out/scan4
bash tools/exp_variants.sh cost_stream cur scan4 cur scan4 > gpurun_out/scan4/variants.log 2>&1
DTB_LIB_PATH=$PWD/build/obj_DTB_COST_SCAN_L4/libdisttrain_b200.so timeout 900 \
  python -m pytest tests -q -m gpu -x > gpurun_out/scan4/tests.log 2>&1
echo done
