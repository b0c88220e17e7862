mkdir -p gpurun_out/small
for S in 8388608 4194304; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/small/launches_$S.csv python bench.py --steps 1 --warmup 3 --no-extras --samples $S > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --samples $S > gpurun_out/small/bench_$S.json 2>/dev/null
done
echo done
