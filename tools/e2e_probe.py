"""Times bench.py's end-to-end leg alone (profiling helper, not part of the
product): dtb_reorder_stream over the 16M-sample mixed stream (BASELINE
config 4) from pinned host buffers, results back to pinned host buffers.
Use DTB_LIB_PATH to time an experiment build."""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import bench as B
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200 import native
    from paper_2408_04275_b200.workload import synth_stream
    model, cluster, book, plan = B.workload()
    plan_c = plan.to_c()
    pl = native.planner(0)
    lib = pl.lib
    cm = pl.cost_model(model, cluster, book)
    mode = A.ReorderMode(1, 0, 0)
    nb = B.STREAM // B.BS
    s = synth_stream(B.STREAM, seed=1000, family="mixed")
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    h = [pin(s.image_offsets), pin(s.image_tokens), pin(s.audio_offsets), pin(s.audio_tokens)]
    I32 = C.POINTER(C.c_int32)
    hs = A.Samples(B.STREAM, None, *[C.cast(x.data_ptr(), I32) for x in h])
    outs = [torch.empty(B.STREAM, dtype=torch.int32).pin_memory(),
            torch.empty(nb * B.DP, dtype=torch.float64).pin_memory(),
            torch.empty(nb * B.DP, dtype=torch.float64).pin_memory(),
            torch.empty(nb, dtype=torch.float64).pin_memory(),
            torch.empty(nb, dtype=torch.float64).pin_memory(),
            torch.empty(nb, dtype=torch.uint8).pin_memory()]
    P = lambda t, ct: C.cast(t.data_ptr(), C.POINTER(ct))

    def call():
        pl._check(lib.reorder_stream(pl.ctx, cm.h, C.byref(plan_c), C.byref(mode), C.byref(hs), nb,
                                     P(outs[0], C.c_int32), P(outs[1], C.c_double),
                                     P(outs[2], C.c_double), P(outs[3], C.c_double),
                                     P(outs[4], C.c_double), P(outs[5], C.c_uint8)))
    call()
    call()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    h2d = sum(x.numel() * 4 for x in h)
    med = float(np.median(ts))
    print(json.dumps({"lib": os.environ.get("DTB_LIB_PATH", "product"), "ms_median": med * 1e3,
                      "ms_min": min(ts) * 1e3, "samples_per_s": B.STREAM / med,
                      "h2d_GBps_equiv": h2d / med / 1e9}))


if __name__ == "__main__":
    main()
