mkdir -p gpurun_out/inter2
timeout 900 python -m pytest tests -q -m gpu -x -k "default or inter or c2 or stream" > gpurun_out/inter2/tests.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:"inter_tok_kernel" -c 2 --csv --log-file gpurun_out/inter2/inter.csv python tools/step_once.py reorder --inter 1 > /dev/null 2>&1
echo done
