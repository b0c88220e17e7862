mkdir -p gpurun_out/inter3
for v in obj obj_DTB_INTER_CARVEOUT100 obj_DTB_INTER_CARVEOUT80; do
  L=paper_2408_04275_b200/libdisttrain_b200.so
  [ "$v" != obj ] && L=build/$v/libdisttrain_b200.so
  DTB_LIB_PATH=$PWD/$L timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"inter_tok_kernel" -c 1 --csv --log-file gpurun_out/inter3/$v.csv python tools/step_once.py reorder --inter 1 > /dev/null 2>&1
done
echo done
