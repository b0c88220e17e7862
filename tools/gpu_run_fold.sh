#!/bin/bash
# The cost pass finalizing each batch in its last chunk's CTA (fold) vs the
# separate finalize kernel (nofold): parity (product + bounds-check builds),
# then step time and launch times.
mkdir -p gpurun_out/fold
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/fold/tests.log 2>&1
DTB_LIB_PATH=$PWD/build/obj_DTB_DEBUG_CHECKS/libdisttrain_b200.so timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/fold/tests_debug.log 2>&1
bash tools/exp_variants.sh "cost_stream|cost_finalize|intra_fused" nofold fold nofold fold > gpurun_out/fold/variants.log 2>&1
for v in nofold fold; do
  cp build/exp/lib_$v.so /tmp/v.so
  DTB_LIB_PATH=/tmp/v.so timeout 300 python tools/probe_intra.py --batches 1024 --check 0 2>&1 | grep "iter 2\|partition kernel" > gpurun_out/fold/probe_$v.log
done
echo done
