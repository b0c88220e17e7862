mkdir -p gpurun_out/r2r
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2r/probe_base.log 2>&1
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 --family dense > gpurun_out/r2r/probe_dense.log 2>&1
for v in obj_DTB_COST_PERSIST1_DTB_COST_T256_DTB_COST_PPS4 obj_DTB_COST_PERSIST1_DTB_COST_T256_DTB_COST_PPS5; do
  E=$PWD/build/$v/libdisttrain_b200.so
  DTB_LIB_PATH=$E timeout 300 python tools/probe_intra.py --batches 1024 --check 2 > gpurun_out/r2r/probe_$v.log 2>&1
  DTB_LIB_PATH=$E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cost_stream -c 3 --csv --log-file gpurun_out/r2r/k0_$v.csv python tools/probe_intra.py --batches 1024 --check 0 > /dev/null 2>&1
done
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2r/gpu_tests.log 2>&1
echo done
