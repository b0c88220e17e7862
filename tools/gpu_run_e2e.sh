#!/bin/bash
# e2e copy-pipeline granularity (DTB_E2E_CHUNKS) and K0 occupancy variants.
mkdir -p gpurun_out/e2e
for v in obj obj_DTB_E2E_CHUNKS16 obj_DTB_E2E_CHUNKS32 obj; do
  L=$PWD/build/$v/libdisttrain_b200.so; [ $v = obj ] && L=$PWD/paper_2408_04275_b200/libdisttrain_b200.so
  DTB_LIB_PATH=$L timeout 300 python tools/e2e_probe.py >> gpurun_out/e2e/e2e.log 2>> gpurun_out/e2e/e2e.err
done
bash tools/exp_variants.sh cost_stream lean occ11 lean occ11 > gpurun_out/e2e/variants.log 2>&1
DTB_LIB_PATH=$PWD/build/obj_DTB_COST_TOKQ10_DTB_COST_MINB11/libdisttrain_b200.so timeout 900 \
  python -m pytest tests -q -m gpu -x -k "stream or dense or fullsize or kept" > gpurun_out/e2e/occ11_tests.log 2>&1
echo done
