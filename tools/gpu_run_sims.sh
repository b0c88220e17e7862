mkdir -p gpurun_out/sims
timeout 600 ncu --set full --import-source on --clock-control none -k regex:group_sims_tiled -c 2 -o gpurun_out/sims/sims python tools/step_once.py reorder --inter 0 > gpurun_out/sims/ncu.log 2>&1
echo done
