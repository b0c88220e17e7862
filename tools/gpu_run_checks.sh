# The GPU suite and the probes against the DTB_DEBUG_CHECKS build (device
# bounds checks that trap on failure; the pool has no compute-sanitizer).
mkdir -p gpurun_out/checks
L=$PWD/build/obj_DTB_DEBUG_CHECKS/libdisttrain_b200.so
DTB_LIB_PATH=$L timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/checks/gpu_tests.log 2>&1
DTB_LIB_PATH=$L timeout 300 python tools/probe_intra.py --batches 1024 --check 2 > gpurun_out/checks/probe_mixed.log 2>&1
DTB_LIB_PATH=$L timeout 300 python tools/probe_intra.py --batches 1024 --check 2 --family dense > gpurun_out/checks/probe_dense.log 2>&1
DTB_LIB_PATH=$L timeout 300 python tools/probe_intra.py --batches 1024 --check 2 --order 1 > gpurun_out/checks/probe_desc.log 2>&1
echo done
