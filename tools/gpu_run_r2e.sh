mkdir -p gpurun_out/r2e
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/r2e/launches.csv python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2e/ncu_l.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cost_stream|intra_fused" -c 2 -o gpurun_out/r2e/sp -f python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/r2e/ncu.log 2>&1
echo done
