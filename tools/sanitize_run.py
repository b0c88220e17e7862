"""Small end-to-end workload for compute-sanitizer (racecheck / synccheck /
memcheck): the reorder stream in every route — histogram path (mixed),
kept path (dense), descending order, default mode with the compiled inter
layouts and the warp-per-problem inter (p = 14), a batch beyond the fused
limits, tiny batches — and a small orchestration search.  Debug tool."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import helpers as H
    from paper_2408_04275_b200 import native
    from paper_2408_04275_b200.api import stats_to_c
    from paper_2408_04275_b200.workload import synth_stream
    pl = native.planner(0)
    model, cluster, book = H.desk_model(), H.desk_cluster(1172), H.desk_book()
    cm = pl.cost_model(model, cluster, book)
    cases = [((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384, 2, "mixed", False, 0),
             ((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384, 2, "dense", False, 0),
             ((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384, 1, "mixed", False, 1),
             ((1, 8, 1), (1, 8, 2), (1, 8, 1), 1024, 2, "mixed", True, 0),
             ((1, 4, 2), (1, 4, 9), (1, 4, 3), 1024, 1, "dense", True, 0),
             ((1, 64, 1), (1, 64, 2), (1, 64, 1), 20000, 1, "mixed", False, 0),
             ((1, 1, 1), (1, 1, 2), (1, 1, 1), 32, 16, "skewed", True, 0)]
    for e, b, g, bs, nb, fam, inter, order in cases:
        plan = H.plan(e, b, g, bs)
        s = synth_stream(nb * bs, seed=3, family=fam)
        pl.reorder_stream(cm, plan, s, nb, inter=inter, sort_order=order)
        print("ok", bs, nb, fam, inter, order, flush=True)
    st = stats_to_c(model.seq_len, 1000.0, 1000.0)
    pl.model_orchestration(pl.cost_model(model, H.desk_cluster(64), book), st, 64)
    print("ok search", flush=True)


if __name__ == "__main__":
    main()
