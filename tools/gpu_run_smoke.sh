#!/bin/bash
# the driver's smoke() and the GPU suite on a box
mkdir -p gpurun_out/smoke
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke/smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/smoke/tests.log 2>&1
echo done
