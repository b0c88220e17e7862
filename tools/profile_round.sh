#!/bin/bash
# Round profiling recipe (runs on the GPU box; see /opt/skills/guides/B200_PROFILING.md):
#  1. the bench exits 0 without ncu;
#  2. a launch list of one bench step (per-launch durations, clocks not locked);
#  3. one `--set full` capture of each sort/partition kernel and of the
#     simulation kernel, with source correlation (compiled -lineinfo).
set -e
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/prof_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extras \
    > gpurun_out/prof_ncu_launch.log 2>&1
for k in token_keys intra_fused group_sims_tiled; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 0 --no-extras \
      > gpurun_out/prof_ncu_$k.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:inter_tok -c 1 \
    -o gpurun_out/full_inter_tok -f python bench.py --steps 1 --warmup 0 \
    > gpurun_out/prof_ncu_inter.log 2>&1 || true
echo profile-done
