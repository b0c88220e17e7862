#!/bin/bash
# Times library variants build/exp/lib_<v>.so in place of the product library:
# bench ms_per_step and the per-kernel ncu launch times of one step.
# usage: tools/exp_variants.sh <kernel-regex> v1 v2 ...
K=$1; shift
cp paper_2408_04275_b200/libdisttrain_b200.so /tmp/orig.so
for v in "$@"; do
  cp build/exp/lib_$v.so paper_2408_04275_b200/libdisttrain_b200.so
  echo "== $v"
  python bench.py --steps 10 --warmup 3 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ms_per_step', d['ms_per_step'])"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K -c 4 --csv python bench.py --steps 1 --warmup 1 --no-extras 2>/dev/null | grep -v '^{' | awk -F'","' 'NR>1{print $NF, substr($5,1,60)}'
done
cp /tmp/orig.so paper_2408_04275_b200/libdisttrain_b200.so
