cp paper_2408_04275_b200/libdisttrain_b200.so /tmp/orig.so
for v in orig exp1 exp2; do
  if [ $v != orig ]; then cp build/exp/lib_$v.so paper_2408_04275_b200/libdisttrain_b200.so; fi
  echo "== $v"
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:group_sims -c 2 --csv python bench.py --steps 1 --warmup 0 --no-extras 2>/dev/null | grep group_sims | awk -F'","' '{print $NF}'
done
cp /tmp/orig.so paper_2408_04275_b200/libdisttrain_b200.so
