"""BASELINE config 5 probe: model_orchestration on the 72B MLLM / 1,172-GPU
cluster at BS 16,384, then disaggregated_reorder of the 16M-sample stream
with the CHOSEN plan.  Checks the chosen plan and sampled batches against the
compiled reference (oracle/_ref) and times both legs on the device.  Debug
tool; not part of the product path."""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=1024)
    ap.add_argument("--check", type=int, default=2)
    ap.add_argument("--inter-batches", type=int, default=1)
    ap.add_argument("--inter-check", type=int, default=0)
    args = ap.parse_args()
    import helpers as H
    import oracle
    from paper_2408_04275_b200 import native
    from paper_2408_04275_b200.api import stats_to_c
    from paper_2408_04275_b200.workload import synth_stream

    pl = native.planner(0)
    ref = oracle.ref()
    m, cl, bk = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
    st = stats_to_c(m.seq_len, 2048.0, 2048.0)
    cm, rcm = pl.cost_model(m, cl, bk), ref.cost_model(m, cl, bk)
    pl.model_orchestration(cm, st, 16384)
    t0 = time.perf_counter()
    g = pl.model_orchestration(cm, st, 16384)
    t_search = time.perf_counter() - t0
    r = ref.model_orchestration(rcm, st, 16384)
    print("plan", g["best"], "match", g["best"] == r["best"] and g["times"] == r["times"],
          f"search {t_search * 1e3:.2f} ms ({g['candidates_evaluated']} candidates)", flush=True)
    plan = g["best"]
    s = synth_stream(args.batches * 16384, seed=1000, family="mixed")
    for inter, nb in ((False, args.batches), (True, args.inter_batches)):
        sub = s.slice(0, nb * 16384)
        pl.reorder_stream(cm, plan, sub, nb, intra=True, inter=inter)
        t0 = time.perf_counter()
        o = pl.reorder_stream(cm, plan, sub, nb, intra=True, inter=inter)
        dt = time.perf_counter() - t0
        print(f"inter={inter} batches={nb} host-api {dt * 1e3:.2f} ms "
              f"({nb * 16384 / dt / 1e6:.1f} M samples/s)", flush=True)
        nchk = args.check if not inter else args.inter_check
        for b in range(min(nchk, nb)):
            one = s.slice(b * 16384, (b + 1) * 16384)
            t0 = time.perf_counter()
            ro = ref.reorder_stream(rcm, plan, one, 1, intra=True, inter=inter)
            rt = time.perf_counter() - t0
            ok = (np.array_equal(ro["output_order"], o["output_order"][b * 16384:(b + 1) * 16384] - b * 16384)
                  or np.array_equal(ro["output_order"], o["output_order"][b * 16384:(b + 1) * 16384]))
            ok = ok and np.array_equal(ro["t_iter_after"], o["t_iter_after"][b:b + 1]) \
                and np.array_equal(ro["load_after"], o["load_after"][b:b + 1])
            print(f"  batch {b}: bit-exact {ok} (reference {rt:.2f} s)", flush=True)


if __name__ == "__main__":
    main()
