# one-GPU evidence (final): bench (all legs), reference arm, refcheck, launch
# list of one bench step, ncu --set full of the sort/partition path kernels
mkdir -p gpurun_out/f8
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/f8/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f8/bench.json 2> gpurun_out/f8/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f8/bench_ref.json 2> gpurun_out/f8/bench_ref.err
timeout 1200 ./oracle/_ref/refcheck > gpurun_out/f8/refcheck.log 2>&1; echo "rc=$?" >> gpurun_out/f8/refcheck.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/f8/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cost_stream|cost_finalize|intra_fused" -c 3 -o gpurun_out/f8/path python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/f8/ncu_path.log 2>&1
timeout 600 python tools/probe_intra.py --batches 1024 --check 3 > gpurun_out/f8/probe.log 2>&1
timeout 600 python tools/probe_intra.py --batches 1024 --check 3 --family dense > gpurun_out/f8/probe_dense.log 2>&1
timeout 600 python tools/probe_intra.py --batches 1024 --check 3 --order 1 > gpurun_out/f8/probe_desc.log 2>&1
echo done
