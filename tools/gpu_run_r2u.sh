mkdir -p gpurun_out/r2u
B=$PWD/build/obj_DTB_SIM_STAGE0/libdisttrain_b200.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:group_sims -c 4 --csv --log-file gpurun_out/r2u/sims_stage.csv python tools/step_once.py reorder --inter 0 > /dev/null 2>&1
DTB_LIB_PATH=$B timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:group_sims -c 4 --csv --log-file gpurun_out/r2u/sims_base.csv python tools/step_once.py reorder --inter 0 > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x -k "not c5_default" > gpurun_out/r2u/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2u/bench.json 2> gpurun_out/r2u/bench.err
DTB_LIB_PATH=$B timeout 600 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/r2u/bench_base.json 2> gpurun_out/r2u/bench_base.err
echo done
