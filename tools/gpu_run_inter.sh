mkdir -p gpurun_out/inter
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"inter_tok_kernel" -c 1 -o gpurun_out/inter/inter python tools/step_once.py reorder --inter 1 > gpurun_out/inter/ncu.log 2>&1
echo done
