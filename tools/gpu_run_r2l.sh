mkdir -p gpurun_out/r2l
for v in obj obj_DTB_COST_Q512_DTB_COST_MINB16 obj_DTB_COST_Q2048_DTB_COST_MINB5; do
  L=paper_2408_04275_b200/libdisttrain_b200.so
  [ "$v" != obj ] && L=build/$v/libdisttrain_b200.so
  DTB_LIB_PATH=$PWD/$L timeout 300 python tools/probe_intra.py --batches 1024 --check 2 > gpurun_out/r2l/probe_$v.log 2>&1
  DTB_LIB_PATH=$PWD/$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cost_stream -c 3 --csv --log-file gpurun_out/r2l/k0_$v.csv python tools/probe_intra.py --batches 1024 --check 0 > /dev/null 2>&1
done
echo done
