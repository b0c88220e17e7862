"""Probe the fused intra kernel on the B200: per-phase timings (globaltimer
stamps of CTA thread 0) over a stream, plus bit-exact spot checks of sampled
batches against the oracle.  Debug tool; not part of the product path."""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=128)
    ap.add_argument("--bs", type=int, default=16384)
    ap.add_argument("--dp", type=int, default=128)
    ap.add_argument("--check", type=int, default=4)
    ap.add_argument("--order", type=int, default=0)
    ap.add_argument("--family", default="mixed")
    args = ap.parse_args()
    import torch
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200 import native
    from paper_2408_04275_b200.workload import synth_stream

    pl = native.planner(0)
    lib = pl.lib
    fn = lib.lib.dtb_debug_intra_stream_prof_dev
    fn.restype = C.c_int32
    fn.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.POINTER(A.Samples), C.c_int64,
                   C.c_void_p, C.c_void_p, C.c_void_p]
    t0 = time.time()
    s = synth_stream(args.batches * args.bs, seed=11, family=args.family)
    print(f"synth {time.time() - t0:.1f}s", flush=True)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d = [dev(s.image_offsets), dev(s.image_tokens), dev(s.audio_offsets), dev(s.audio_tokens)]
    ds = A.Samples(s.n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in d])
    out = torch.empty(s.n, dtype=torch.int32, device="cuda")
    prof = torch.zeros(args.batches * 64, dtype=torch.int64, device="cuda")
    for it in range(3):
        prof.zero_()
        prof[62] = -1  # atomicMin slot (unsigned max)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pl._check(fn(pl.ctx, args.bs, args.dp, args.order, C.byref(ds), args.batches,
                     C.c_void_p(out.data_ptr()), C.c_void_p(prof.data_ptr()), None))
        e1.record()
        torch.cuda.synchronize()
        print(f"iter {it}: kernel {e0.elapsed_time(e1):.3f} ms", flush=True)
    p = prof.view(args.batches, 64).cpu().numpy().astype(np.float64)
    entry, leave = p[0, 62], p[0, 63]
    if leave > entry:
        print(f"  partition kernel: first CTA entry -> last CTA exit {(leave - entry) / 1e3:.1f} us")
    p[0, 62] = p[0, 63] = 0
    done = p[:, 0] > 0  # batches the partition kernel processed
    print(f"processed by the partition kernel: {int(done.sum())} of {args.batches}")
    if done.any():
        p0 = p[done, 0].min()
        if entry > 0:
            print(f"  kernel entry (CTA 0) -> first start {(p0 - entry) / 1e3:.1f} us")
        print(f"  first start -> last start {(p[done, 0].max() - p0) / 1e3:.1f} us, "
              f"first start -> last end {(p[done, 5].max() - p0) / 1e3:.1f} us")
        p = p[done]
    names = ["load+cost", "sort", "greedy", "partition+decide", "outputs"]
    span = (p[:, 5] - p[:, 0]) / 1e3
    print(f"per-CTA span us: median {np.median(span):.1f} max {span.max():.1f}")
    for k, nm in enumerate(names):
        dt = (p[:, k + 1] - p[:, k]) / 1e3
        print(f"  {nm:18s} median {np.median(dt):8.1f} us  max {dt.max():8.1f}")
    pi = prof.view(args.batches, 64).cpu().numpy()[done] if done.any() else prof.view(args.batches, 64).cpu().numpy()
    z = (p[:, 6] - p[:, 2]) / 1e3
    ok = pi[:, 6] > 0
    if ok.any():
        print(f"  greedy: zero run median {np.median(z[ok]):.1f} us; rest "
              f"{np.median(((p[:, 3] - p[:, 6]) / 1e3)[ok]):.1f} us")
    cnt = pi[:, 7]
    print(f"  greedy rounds: full segments median {np.median(cnt >> 32):.0f}, "
          f"general median {np.median(cnt & 0xffffffff):.0f} max {(cnt & 0xffffffff).max()}")
    st = p[:, 8:56].reshape(len(p), 16, 3)
    if (st[:, 0, 0] > 0).any():
        prev = np.concatenate([p[:, :1], st[:, :-1, 2]], axis=1)  # previous stage end
        wait = (st[:, :, 0] - prev) / 1e3
        pref = (st[:, :, 1] - st[:, :, 0]) / 1e3
        loop = (st[:, :, 2] - st[:, :, 1]) / 1e3
        for k in (0, 1, 2, 8, 15):
            print(f"  stage {k:2d}: wait median {np.median(wait[:, k]):6.2f} us, prefix "
                  f"{np.median(pref[:, k]):6.2f}, samples+sync {np.median(loop[:, k]):6.2f}")
    if (p[:, 57] > 0).any():
        rel = lambda k: (p[:, k] - p[:, 0]) / 1e3
        print(f"  pair: peer sort done median {np.median(rel(57)):.1f} max {rel(57).max():.1f} us; "
              f"first cluster sync {np.median(rel(58)):.1f} / {rel(58).max():.1f}; "
              f"second {np.median(rel(59)):.1f} / {rel(59).max():.1f} (from batch start)")
        kp = pi[:, 0] > 0
        gap = rel(59) - rel(58)
        for i in np.argsort(-gap)[:4]:  # the kept batches: rank 1 writes the order in between
            print(f"    batch row {i}: first sync {rel(58)[i]:.1f}, second {rel(59)[i]:.1f}, "
                  f"gap {gap[i]:.1f} us, outputs end {rel(5)[i]:.1f}"
                  + (f", kept order written {rel(61)[i]:.1f} -> {rel(60)[i]:.1f}" if p[i, 60] > 0 else ""))
    ks = p[:, 56:61] * 0
    okk = ks[:, 0] > 0
    if okk.any():
        names_k = ["heavy ids", "counts", "walk", "light sort"]
        print(f"  kept scatter ({okk.sum()} batches):", ", ".join(
            f"{nm} {np.median((ks[okk, k + 1] - ks[okk, k]) / 1e3):.1f}" for k, nm in enumerate(names_k)))
    if args.check:
        import oracle
        import helpers as H
        ora, kind = oracle.best()
        model, cluster, book = H.desk_model(), H.desk_cluster(1172), H.desk_book()
        co = ora.cost_model(model, cluster, book)
        plan = H.plan((1, args.dp, 1), (1, args.dp, 2), (1, args.dp, 1), args.bs)
        got = out.cpu().numpy().reshape(args.batches, args.bs)
        rng = np.random.default_rng(0)
        for bidx in sorted(rng.choice(args.batches, min(args.check, args.batches), replace=False)):
            r = ora.disaggregated_reorder(co, plan, s.slice(bidx * args.bs, (bidx + 1) * args.bs),
                                          inter=False, sort_order=args.order)
            ok = np.array_equal(r.output_order, got[bidx])
            print(f"  batch {bidx}: {'bit-exact' if ok else 'MISMATCH'} vs {kind}", flush=True)


if __name__ == "__main__":
    main()
