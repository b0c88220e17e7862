mkdir -p gpurun_out/r2c
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"intra_fused" -c 1 -o gpurun_out/r2c/sp -f python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2c/ncu.log 2>&1
echo done
