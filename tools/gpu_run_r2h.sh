mkdir -p gpurun_out/r2h
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cost_stream" -c 1 -o gpurun_out/r2h/k0 -f python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2h/ncu.log 2>&1
echo done
