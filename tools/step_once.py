"""One call of a hot-path entry point for ncu captures (profiling helper, not
part of the product): `reorder` = dtb_reorder_stream_dev over the 16M-sample
mixed stream (BASELINE config 4) in intra or default mode; `search` =
model_orchestration for BASELINE config 3.  Runs `--reps` calls after one
warm-up call."""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["reorder", "search"])
    ap.add_argument("--inter", type=int, default=0)
    ap.add_argument("--batches", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import helpers as H
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200 import native
    from paper_2408_04275_b200.api import stats_to_c
    pl = native.planner(0)
    lib = pl.lib
    if args.what == "search":
        m, cl, bk = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
        st = stats_to_c(m.seq_len, 2048.0, 2048.0)
        cm = pl.cost_model(m, cl, bk)
        res = A.OrchestrationResult()
        for _ in range(1 + args.reps):
            pl._check(lib.model_orchestration(pl.ctx, cm.h, C.byref(st), 1920, 1, C.byref(res), None, 0))
        print("candidates", res.candidates_evaluated)
        return
    from paper_2408_04275_b200.workload import synth_stream
    bs, dp, nb = 16384, 128, args.batches
    s = synth_stream(nb * bs, seed=1000, family="mixed")
    cm = pl.cost_model(H.desk_model(), H.desk_cluster(1172), H.desk_book())
    plan = H.plan((1, dp, 1), (1, dp, 2), (1, dp, 1), bs).to_c()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d = [dev(s.image_offsets), dev(s.image_tokens), dev(s.audio_offsets), dev(s.audio_tokens)]
    ds = A.Samples(s.n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in d])
    f64 = lambda k: torch.zeros(k, dtype=torch.float64, device="cuda")
    out = [torch.empty(s.n, dtype=torch.int32, device="cuda"), f64(nb * dp), f64(nb * dp),
           f64(nb), f64(nb), torch.zeros(nb, dtype=torch.uint8, device="cuda")]
    mode = A.ReorderMode(1, args.inter, 0)
    sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(1 + args.reps):
        pl._check(lib.reorder_stream_dev(pl.ctx, cm.h, C.byref(plan), C.byref(mode), C.byref(ds), nb,
                                         *[C.c_void_p(x.data_ptr()) for x in out], sh))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
