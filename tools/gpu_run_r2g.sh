mkdir -p gpurun_out/r2g
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"intra_fused" -c 1 -o gpurun_out/r2g/dense -f python tools/probe_intra.py --batches 1024 --check 0 --family dense > gpurun_out/r2g/ncu.log 2>&1
echo done
