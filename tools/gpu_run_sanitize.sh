mkdir -p gpurun_out/r2s
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2s/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2s/$tool.log
done
echo done
