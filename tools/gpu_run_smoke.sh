#!/bin/bash
mkdir -p gpurun_out/smoke
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke/smoke.log
echo done
