# one-GPU evidence for profiles/: bench (all legs), reference arm, refcheck,
# launch list of one bench step, ncu --set full of K0 / finalize / K1
mkdir -p gpurun_out/f1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f1/bench.json 2> gpurun_out/f1/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f1/bench_ref.json 2> gpurun_out/f1/bench_ref.err
timeout 1200 ./oracle/_ref/refcheck > gpurun_out/f1/refcheck.log 2>&1; echo "rc=$?" >> gpurun_out/f1/refcheck.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/f1/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cost_stream|cost_finalize|intra_fused" -c 3 -o gpurun_out/f1/path python tools/probe_intra.py --batches 1024 --check 0 > gpurun_out/f1/ncu_path.log 2>&1
echo done
