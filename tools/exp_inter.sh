#!/bin/bash
# Times inter-reorder library variants build/exp/lib_<v>.so (device path,
# tools/run_inter_dev.py) in place of the product library.
cp paper_2408_04275_b200/libdisttrain_b200.so /tmp/orig.so
for v in "$@"; do
  cp build/exp/lib_$v.so paper_2408_04275_b200/libdisttrain_b200.so
  echo "== $v"
  python tools/run_inter_dev.py 2>&1 | tail -1
done
cp /tmp/orig.so paper_2408_04275_b200/libdisttrain_b200.so
