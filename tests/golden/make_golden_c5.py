"""Generates tests/golden/c5_default.npz: the UNMODIFIED reference
(oracle/_ref, compiled from /root/reference) on BASELINE config 5 in default
mode — model_orchestration of the 72B MLLM on 1,172 GPUs at BS 16,384, then
disaggregated_reorder (intra + inter) of one 16K-sample global batch of the
mixed stream (seed 1000) with the CHOSEN plan (DP 16, PP 1/71/7: l = 1,024,
p = 79).  One reference call takes ~2 minutes on one core, so the GPU test
(tests/test_gpu_fullsize.py) replays this fixture instead of re-running it.

    python tests/golden/make_golden_c5.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def c5_inputs():
    import helpers as H
    from paper_2408_04275_b200.api import stats_to_c
    from paper_2408_04275_b200.workload import synth_stream
    m, cl, bk = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
    return m, cl, bk, stats_to_c(m.seq_len, 2048.0, 2048.0), synth_stream(16384, seed=1000,
                                                                           family="mixed")


def main():
    import oracle
    if not oracle.ref_available():
        oracle.build(ref=True)
    ref = oracle.ref()
    m, cl, bk, st, s = c5_inputs()
    co = ref.cost_model(m, cl, bk)
    res = ref.model_orchestration(co, st, 16384)
    best = res["best"]
    r = ref.reorder_stream(co, best, s, 1, inter=True)
    pp = [best.encoder.pp, best.backbone.pp, best.generator.pp]
    dp = [best.encoder.dp, best.backbone.dp, best.generator.dp]
    tp = [best.encoder.tp, best.backbone.tp, best.generator.tp]
    np.savez_compressed(os.path.join(HERE, "c5_default.npz"), tp=tp, dp=dp, pp=pp,
                        vpp=best.vpp, times=np.array(res["times"]),
                        **{k: np.asarray(v) for k, v in r.items()})
    print(best, {k: np.asarray(v).shape for k, v in r.items()})


if __name__ == "__main__":
    main()
