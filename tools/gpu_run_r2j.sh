mkdir -p gpurun_out/r2j
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
F=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"cost_stream|cost_finalize|intra_fused" -c 6 --csv --log-file gpurun_out/r2j/traffic.csv python tools/probe_intra.py --batches 1024 --check 0 > /dev/null 2>&1
timeout 600 ncu --metrics $F --clock-control none -c 40 --csv --log-file gpurun_out/r2j/fp64_search.csv python tools/step_once.py search > /dev/null 2>&1
timeout 600 ncu --metrics $F --clock-control none -k regex:"group_sims|inter_tok|inter_warp" -c 8 --csv --log-file gpurun_out/r2j/fp64_reorder.csv python tools/step_once.py reorder --inter 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cost_stream" -s 1 -c 1 -o gpurun_out/r2j/k0 python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2j/ncu_k0.log 2>&1
echo done
