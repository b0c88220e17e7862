#!/bin/bash
# Cost pass: closing boundary gathers passed by a shuffle (DTB_COST_SHFL=1)
# vs one gather per lane (=0); parity of the shuffle build.
mkdir -p gpurun_out/shfl
bash tools/exp_variants.sh cost_stream noshfl shfl noshfl shfl > gpurun_out/shfl/variants.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/shfl/tests.log 2>&1
echo done
