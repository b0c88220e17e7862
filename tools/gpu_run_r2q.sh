mkdir -p gpurun_out/r2q
E=$PWD/build/obj_DTB_COST_PERSIST1/libdisttrain_b200.so
timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2q/probe_base.log 2>&1
DTB_LIB_PATH=$E timeout 300 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/r2q/probe_persist.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cost_stream -c 3 --csv --log-file gpurun_out/r2q/k0_base.csv python tools/probe_intra.py --batches 1024 --check 0 > /dev/null 2>&1
DTB_LIB_PATH=$E timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cost_stream -c 3 --csv --log-file gpurun_out/r2q/k0_persist.csv python tools/probe_intra.py --batches 1024 --check 0 > /dev/null 2>&1
DTB_LIB_PATH=$E timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2q/gpu_tests_persist.log 2>&1
echo done
