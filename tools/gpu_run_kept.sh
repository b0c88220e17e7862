#!/bin/bash
# Kept-batch simulation kernel (group_sims_kept) vs the tiled kernel
# (DTB_NO_KEPT_SIMS build): parity, then step time and launch list at the full,
# half and quarter stream (the quarter is one rank's range at N = 4).
mkdir -p gpurun_out/kept
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/kept/gpu_tests.log 2>&1
for v in product nokept; do
  L=$PWD/paper_2408_04275_b200/libdisttrain_b200.so; [ $v = nokept ] && L=$PWD/build/obj_DTB_NO_KEPT_SIMS/libdisttrain_b200.so
  for S in 16777216 4194304; do
    DTB_LIB_PATH=$L timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --samples $S > gpurun_out/kept/bench_${v}_$S.json 2>/dev/null
    DTB_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/kept/launches_${v}_$S.csv python bench.py --steps 1 --warmup 3 --no-extras --samples $S > /dev/null 2>&1
  done
done
echo done
