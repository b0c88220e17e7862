"""Benchmark: DistTrain reorder hot path on B200 (BASELINE.json config 4).

Workload: a 16,777,216-sample synthetic image+audio stream (variable
resolution -> patch tokens, audio clips) in global batches of 16,384, plan
DP_lm = DP_me = DP_mg = 128, PP 1/2/1 (l = 128 microbatches per pipeline), the
reference's desk-shaped cost profile (proj/tests/support/configs.hpp:79-102).
One step = `disaggregated_reorder` (src/reorder.cpp:319-396) over every
global batch of the stream with ReorderMode{intra=true, inter=false}:
per-sample cost, stable sort, greedy equal-count partition, keep-if-no-worse,
group loads and both simulated iteration times -- the sort/partition path
the north_star's HBM target names.  The full default mode (intra + inter)
and the orchestration search (BASELINE config 3) are measured too and
reported under "modes" / "search".

N GPUs (torchrun): STRONG scaling — ONE 16M-sample stream split by
global-batch range (dtb_shard_range), each rank reorders its range and the
library stores every rank's ordering into every rank's replica over NVLink
(dtb_reorder_stream_shard_dev: CUDA-IPC peer stores on a side stream that
overlaps the simulations, device flag barrier); `value` = 16M samples / the
max-over-ranks device time of that call, with the whole ordering present on
every rank.  "weak" (each rank its own 16M stream, no exchange) is an extra.

--impl reference: the reference's own CPU implementation (oracle/_ref,
compiled from the reference sources; the C restatement if absent) on all
host threads, on a bounded sample of the same stream.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

BS = 16384
DP = 128
STREAM = 1 << 24
METRIC = "reordered samples/s (disaggregated_reorder, 16M-sample stream, BS 16K, DP 128)"
# cost_stream, cost_finalize, intra_fused, cost_table, 2x group_sims, 2x t_iter_reduce
LAUNCHES_INTRA_STEP = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=STREAM)
    ap.add_argument("--no-extras", action="store_true", help="skip modes/e2e/cpu/search legs")
    return ap.parse_args()


def dist_init():
    # stdout carries exactly one JSON line: NCCL's INFO/VERSION banner
    # ("NCCL version ...") would precede it on rank 0
    if not os.environ.get("DTB_KEEP_NCCL_DEBUG"):
        # NCCL logs (incl. its "NCCL version" banner, printed at WARN too) go
        # to stderr: stdout carries exactly one JSON line
        os.environ["NCCL_DEBUG"] = "WARN"
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload():
    import helpers as H
    model, cluster, book = H.desk_model(), H.desk_cluster(1172), H.desk_book()
    plan = H.plan((1, DP, 1), (1, DP, 2), (1, DP, 1), BS)
    return model, cluster, book, plan


def search_workload():
    """BASELINE config 3: 72B MLLM on 1172 A800-like GPUs, BS 1920."""
    import helpers as H
    from paper_2408_04275_b200.api import stats_to_c
    model = H.mllm72b_model()
    return model, H.a800_cluster(1172), H.mllm72b_book(), 1920, stats_to_c(model.seq_len, 2048.0,
                                                                          2048.0)


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, idx):
        self.idx, self.proc = idx, None
        self.path = f"/tmp/dtb_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.2)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r]
        except Exception:
            return None
        if not rows:
            return None
        num = lambda s: float(s) if s.strip().replace(".", "").isdigit() else None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        mx = [num(r[1]) for r in rows if len(r) > 1 and num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def cpu_reference(samples, plan_c, mode, n_batches, steps, warmup, threads, cm, bs=BS):
    """The reference's own disaggregated_reorder (oracle/_ref) over n_batches
    global batches, fanned out over `threads` host threads.  Samples are
    converted to std::vector<Sample> outside the timed region."""
    import oracle
    pl, kind = oracle.best()
    lib = pl.lib
    sub = samples.slice(0, n_batches * bs)
    s = sub.to_c()
    h = C.c_void_p()
    pl._check(lib.stream_prepare(C.byref(s), n_batches, C.byref(h)))
    lib.set_threads(threads)
    ocm = pl.cost_model(*cm)
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        pl._check(lib.stream_run(h, ocm.h, C.byref(plan_c), C.byref(mode), 0, n_batches,
                                 None, None, None, None, None))
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    lib.stream_destroy(h)
    return kind, times


def cpu_search(threads):
    """model_orchestration on the reference (multi-threaded fan-out)."""
    import oracle
    from paper_2408_04275_b200 import _capi as A
    pl, kind = oracle.best()
    model, cluster, book, bs, stats = search_workload()
    cm = pl.cost_model(model, cluster, book)
    res = A.OrchestrationResult()
    if pl.lib.has("model_orchestration_mt"):
        pl.lib.set_threads(threads)
        t0 = time.perf_counter()
        pl._check(pl.lib.model_orchestration_mt(pl.ctx, cm.h, C.byref(stats), bs, 1, C.byref(res)))
    else:
        threads = 1
        t0 = time.perf_counter()
        pl._check(pl.lib.model_orchestration(pl.ctx, cm.h, C.byref(stats), bs, 1, C.byref(res),
                                             None, 0))
    dt = time.perf_counter() - t0
    return kind, threads, res.candidates_evaluated / dt, dt, res


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def traffic_from_profiles():
    """dram bytes per launch of the sort/partition kernels from the committed
    ncu --set full summary (profiles/), if present."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return d
    except Exception:
        return None


def reference_arm(args, model, cluster, book, plan_c):
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200.workload import synth_stream
    threads = os.cpu_count() or 1
    n_total = args.samples // BS
    sample_batches = max(1, min(n_total, 2 * threads))
    samples = synth_stream(sample_batches * BS, seed=1000, family="mixed")
    kind, times = cpu_reference(samples, plan_c, A.ReorderMode(1, 0, 0), sample_batches,
                                max(1, min(args.steps, 100)), args.warmup, threads,
                                (model, cluster, book))
    t = float(np.median(times))
    v = sample_batches * BS / t
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64 tokens / f64 loads and stage times",
            "data": "synthetic (PCG64 mixed image+audio stream)",
            "config": {"workload": "BASELINE config 4: global batch 16384, DP 128, PP 1/2/1, "
                                   "ReorderMode{intra} (bounded CPU sample of the stream)",
                       "global_batch": BS, "dp": DP, "sample_batches": sample_batches},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": kind,
                             "cpu_model": cpu_model(),
                             "sample": f"{sample_batches} global batches x {BS} samples, "
                                       f"std::thread fan-out over batches"},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank, world, local = dist_init()
    model, cluster, book, plan = workload()
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200 import shard
    from paper_2408_04275_b200.workload import synth_stream

    plan_c = plan.to_c()
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args, model, cluster, book, plan_c)), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    from paper_2408_04275_b200 import native
    pl = native.planner(local)
    lib = pl.lib
    cm = pl.cost_model(model, cluster, book)
    mode_intra, mode_both = A.ReorderMode(1, 0, 0), A.ReorderMode(1, 1, 0)

    # ONE stream of 16M samples (1,024 global batches); at N > 1 every rank
    # holds it and reorders its batch range (strong scaling)
    my_batches = args.samples // BS
    samples = synth_stream(my_batches * BS, seed=1000, family="mixed")
    n = samples.n
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_csr = [dev(samples.image_offsets), dev(samples.image_tokens), dev(samples.audio_offsets),
             dev(samples.audio_tokens)]
    ds = A.Samples(n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in d_csr])
    out_order = torch.empty(n, dtype=torch.int32, device="cuda")
    lb = torch.empty(my_batches * DP, dtype=torch.float64, device="cuda")
    la = torch.empty_like(lb)
    tb = torch.empty(my_batches, dtype=torch.float64, device="cuda")
    ta = torch.empty_like(tb)
    kept = torch.empty(my_batches, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2 (126 MB)
    stream = torch.cuda.Stream()
    sh = C.c_void_p(stream.cuda_stream)
    ptr = lambda t: C.c_void_p(t.data_ptr())

    def step(mode, sub=None, nb=my_batches):
        pl._check(lib.reorder_stream_dev(pl.ctx, cm.h, C.byref(plan_c), C.byref(mode),
                                         C.byref(sub or ds), nb, ptr(out_order), ptr(lb),
                                         ptr(la), ptr(tb), ptr(ta), ptr(kept), sh))

    def sort_partition():
        pl._check(lib.intra_stream_dev(pl.ctx, BS, DP, 0, C.byref(ds), my_batches,
                                       ptr(out_order), ptr(lb), ptr(la), ptr(kept), sh))

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        evs = []
        with torch.cuda.stream(stream):
            for _ in range(steps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                fn()
                e.record(stream)
                evs.append((s, e))
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        return float(np.mean([s.elapsed_time(e) for s, e in evs]))

    group = replica = None
    if world > 1:
        # the library's exchange: every rank's replica of the whole ordering
        import torch.distributed as dist
        replica, handle = pl.peer_buffer_create(n)
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        group = pl.peer_group_open(rank, world, replica, n, handles)

        def headline():
            pl._check(lib.reorder_stream_shard_dev(pl.ctx, cm.h, C.byref(plan_c),
                                                   C.byref(mode_intra), C.byref(ds), my_batches,
                                                   group, ptr(lb), ptr(la), ptr(tb), ptr(ta),
                                                   ptr(kept), sh))
    else:
        def headline():
            step(mode_intra)
    # the same call captured once into a CUDA graph (fixed pointers) and
    # replayed: one launch per step instead of ~10 host-side launches
    graph = C.c_void_p()
    pl._check(lib.reorder_stream_graph_create(pl.ctx, cm.h, C.byref(plan_c), C.byref(mode_intra),
                                              C.byref(ds), my_batches, group, ptr(out_order),
                                              ptr(lb), ptr(la), ptr(tb), ptr(ta), ptr(kept),
                                              C.byref(graph)))

    def headline_graph():
        pl._check(lib.graph_launch(graph, sh))
    ms_direct = max_over_ranks(timed(headline, max(3, args.steps // 2), args.warmup), world)
    with Clocks(local) as clk:
        ms_local = timed(headline_graph, args.steps, args.warmup)
    ms = max_over_ranks(ms_local, world)
    total = my_batches * BS
    first_b, count_b = shard.batch_range(my_batches, rank, world)
    out = {"metric": METRIC, "value": total / (ms / 1e3), "unit": "samples/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "int32 tokens / int64 loads / f64 stage times (u16 sort keys)",
           "data": "synthetic (PCG64 mixed image+audio stream; desk-shaped cost profile)",
           "config": {"workload": "BASELINE config 4: ONE 16M-sample stream, global batch "
                                  "16384, DP 128, PP 1/2/1, disaggregated_reorder "
                                  "ReorderMode{intra}",
                      "samples": total, "samples_per_gpu": count_b * BS, "global_batch": BS,
                      "dp": DP,
                      "parallelism": (f"global-batch-range sharding over {world} GPUs; the "
                                      "whole ordering (u16 in-batch indices) stored into every "
                                      "rank's replica by the library over NVLink (CUDA IPC "
                                      "peer stores + device flag barrier), inside the timed "
                                      "region") if world > 1 else "1 GPU",
                      "l2": "256 MiB buffer written between timed steps (inputs also > L2)"},
           "gpu_launches": LAUNCHES_INTRA_STEP + (1 if world > 1 else 0),
           "launch": "one CUDA graph launch per step (dtb_reorder_stream_graph_create)",
           "ms_per_step_direct_calls": ms_direct}
    clocks = clk.summary()
    if clocks:
        out["clocks"] = clocks

    # ---- roofline of the sort/partition path (cost pass + fused partition)
    sp_local = timed(sort_partition, args.steps, args.warmup)
    n_img, n_aud = len(samples.image_tokens), len(samples.audio_tokens)
    algo = (4 * 2 * (n + my_batches) + 4 * (n_img + n_aud)   # CSR offsets + tokens in
            + 4 * n + 2 * 8 * DP * my_batches + my_batches)  # order + both loads + kept out
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = algo / (sp_local / 1e3) / 1e9
    tr = traffic_from_profiles()
    kernels = ("cost_stream_kernel + cost_finalize_kernel + intra_fused_kernel (sort/partition "
               "path: dtb_intra_stream_dev, its scratch memset included)")
    out["roofline"] = {
        "bound": "hbm", "kernel": kernels,
        "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
        # ncu capture of the 16M stream, scaled to this rank's samples
        "traffic": round(tr["bytes_per_step_16M"] * n / STREAM) if tr else None,
        "algorithmic_bytes_per_launch": algo, "ms_per_launch": sp_local,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650",
        "stream": "mixed (BASELINE config 4): the greedy split loses on most batches"}
    if not args.no_extras and world == 1:
        # descending order (the LPT variant, ReorderMode::sort_order) on the
        # same stream: the averaging bound does not apply, every batch runs
        # the histogram greedy and most keep it
        def sort_partition_desc():
            pl._check(lib.intra_stream_dev(pl.ctx, BS, DP, 1, C.byref(ds), my_batches,
                                           ptr(out_order), ptr(lb), ptr(la), ptr(kept), sh))
        spx = timed(sort_partition_desc, max(3, args.steps // 2), args.warmup)
        ach_x = algo / (spx / 1e3) / 1e9
        out["roofline_descending"] = {
            "bound": "hbm", "kernel": kernels, "achieved": ach_x, "peak": hbm, "unit": "GB/s",
            "frac": ach_x / hbm, "ms_per_launch": spx,
            "stream": f"mixed, descending sort order: greedy split kept on "
                      f"{float(kept.float().mean().item()):.0%} of the batches"}
        # the same path on the dense family (every sample has an image): the
        # greedy split is KEPT on every batch, so the stable sort and the
        # permutation run on all of them
        dense = synth_stream(my_batches * BS, seed=1000, family="dense")
        dd = [dev(dense.image_offsets), dev(dense.image_tokens), dev(dense.audio_offsets),
              dev(dense.audio_tokens)]
        dds = A.Samples(n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in dd])

        def sort_partition_dense():
            pl._check(lib.intra_stream_dev(pl.ctx, BS, DP, 0, C.byref(dds), my_batches,
                                           ptr(out_order), ptr(lb), ptr(la), ptr(kept), sh))
        spd = timed(sort_partition_dense, max(3, args.steps // 2), args.warmup)
        algo_d = (4 * 2 * (n + my_batches) + 4 * (len(dense.image_tokens) + len(dense.audio_tokens))
                  + 4 * n + 2 * 8 * DP * my_batches + my_batches)
        kept_frac = float(kept.float().mean().item())
        ach_d = algo_d / (spd / 1e3) / 1e9
        out["roofline_kept"] = {
            "bound": "hbm", "kernel": kernels, "achieved": ach_d, "peak": hbm, "unit": "GB/s",
            "frac": ach_d / hbm, "algorithmic_bytes_per_launch": algo_d, "ms_per_launch": spd,
            "stream": "dense (mixed with >= 1 image per sample): greedy split kept on "
                      f"{kept_frac:.0%} of the batches"}
        del dd

    if world > 1:
        # weak-scaling extra: every rank reorders the whole stream (no exchange)
        w_ms = max_over_ranks(timed(lambda: step(mode_intra), max(2, args.steps // 2), 1), world)
        out["weak"] = {"samples": total * world, "ms_per_step": w_ms,
                       "value": total * world / (w_ms / 1e3), "unit": "samples/s",
                       "what": "every rank reorders its own copy of the 16M stream; no exchange"}

    if not args.no_extras:
        # e2e on every rank: host CSR (pinned) -> device -> results back,
        # through the public C ABI (dtb_reorder_stream, copy/compute pipelined)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        h_csr = [pin(samples.image_offsets), pin(samples.image_tokens),
                 pin(samples.audio_offsets), pin(samples.audio_tokens)]
        # this rank's batch range of the stream (the whole stream at N = 1):
        # offsets from the range's first sample, absolute into the tokens
        n_sh = count_b * BS
        off = lambda t: C.cast(t.data_ptr() + 4 * first_b * BS, C.POINTER(C.c_int32))
        hs = A.Samples(n_sh, None, off(h_csr[0]), C.cast(h_csr[1].data_ptr(), C.POINTER(C.c_int32)),
                       off(h_csr[2]), C.cast(h_csr[3].data_ptr(), C.POINTER(C.c_int32)))
        h_order = torch.empty(n_sh, dtype=torch.int32).pin_memory()
        h_lb = torch.empty(count_b * DP, dtype=torch.float64).pin_memory()
        h_la = torch.empty_like(h_lb).pin_memory()
        h_tb = torch.empty(count_b, dtype=torch.float64).pin_memory()
        h_ta = torch.empty_like(h_tb).pin_memory()
        h_kept = torch.empty(count_b, dtype=torch.uint8).pin_memory()
        P = lambda t, ct: C.cast(t.data_ptr(), C.POINTER(ct))

        def e2e():
            pl._check(lib.reorder_stream(pl.ctx, cm.h, C.byref(plan_c), C.byref(mode_intra),
                                         C.byref(hs), count_b, P(h_order, C.c_int32),
                                         P(h_lb, C.c_double), P(h_la, C.c_double),
                                         P(h_tb, C.c_double), P(h_ta, C.c_double),
                                         P(h_kept, C.c_uint8)))
        e2e()
        reps = max(3, args.steps // 2)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e()
        e_dt = max_over_ranks((time.perf_counter() - t0) / reps, world)
        io_h, ao_h = samples.image_offsets, samples.audio_offsets
        h2d = 4 * (2 * (n_sh + 1) + int(io_h[(first_b + count_b) * BS] - io_h[first_b * BS]) +
                   int(ao_h[(first_b + count_b) * BS] - ao_h[first_b * BS]))
        d2h = sum(x.numel() * x.element_size() for x in (h_order, h_lb, h_la, h_tb, h_ta, h_kept))
        out["e2e"] = {"value": total / e_dt, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "ms_per_step": e_dt * 1e3,
                      "path": "dtb_reorder_stream (host pointers, pinned; each rank its batch "
                              "range of the one stream; per-rank bytes, max over ranks)"}

    if not args.no_extras and rank == 0 and world == 1:
        # full default mode (intra + inter)
        both_ms = timed(lambda: step(mode_both), max(2, args.steps // 3), 1)
        out["modes"] = {"intra+inter": {"ms_per_step": both_ms,
                                        "value": my_batches * BS / (both_ms / 1e3),
                                        "unit": "samples/s"}}
        # the reference's default mode on a bounded sample (one global batch per
        # host thread, ~1 s per batch on one core)
        thr = os.cpu_count() or 1
        kind_d, times_d = cpu_reference(samples, plan_c, mode_both, min(my_batches, thr), 1, 0, thr,
                                        (model, cluster, book))
        out["modes"]["intra+inter"]["cpu_baseline"] = {
            "value": min(my_batches, thr) * BS / float(np.median(times_d)), "unit": "samples/s",
            "cores": thr, "kind": kind_d, "cpu_model": cpu_model(),
            "sample": f"first {min(my_batches, thr)} global batches x {BS} samples, default mode, "
                      "std::thread fan-out over batches"}
        try:  # FP64 instructions of the step (ncu count) over the measured step time
            fops = json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_ops.json")))
            ks = fops["reorder_default_16M"]["kernels"]
            per = {k: v["dadd"] + v["dmul"] + v["dfma"] for k, v in ks.items()}
            inst = per["inter_tok_kernel"] + per["inter_tok_kernel_redo"] + 2 * per["group_sims_tiled"]
            if my_batches * BS == STREAM:
                ach = inst / (both_ms / 1e3)
                out["modes"]["intra+inter"]["roofline_fp64"] = {
                    "bound": "fp64", "kernel": "inter_tok_kernel (dominant) + 2 x group_sims_tiled",
                    "achieved": ach, "peak": fops["peak_fp64_instr_per_s"], "unit": "FP64 instr/s",
                    "frac": ach / fops["peak_fp64_instr_per_s"], "fp64_instr_per_step": inst,
                    "note": "over the whole step time (a lower bound for the kernels); the FP64 "
                            "pipe is not the limiter: the inter kernel is latency-bound",
                    "counts_source": fops["reorder_default_16M"]["source"]}
        except Exception:
            pass
        # BASELINE config 2: LLaVA-style ViT-L + 7B backbone, PP 1/2/1 (4
        # devices), 32 microbatches per iteration, 10K independent iterations
        # — one global batch of 32 samples per iteration (DP 1), default
        # mode (intra + inter), on the same stream entry point
        import helpers as H
        c2_iters, c2_l = 10000, 32
        c2_model, c2_cluster, c2_book = H.llava_model(), H.a800_cluster(64), H.llava_book()
        c2_cm = pl.cost_model(c2_model, c2_cluster, c2_book)
        c2_plan = H.plan((1, 1, 1), (1, 1, 2), (1, 1, 1), c2_l).to_c()
        c2_s = synth_stream(c2_iters * c2_l, seed=2024, family="skewed")
        c2_d = [dev(c2_s.image_offsets), dev(c2_s.image_tokens), dev(c2_s.audio_offsets),
                dev(c2_s.audio_tokens)]
        c2_ds = A.Samples(c2_s.n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32))
                                           for x in c2_d])
        c2_out = [torch.empty(c2_s.n, dtype=torch.int32, device="cuda")] + \
                 [torch.empty(c2_iters, dtype=torch.float64, device="cuda") for _ in range(4)] + \
                 [torch.empty(c2_iters, dtype=torch.uint8, device="cuda")]

        def c2_step():
            pl._check(lib.reorder_stream_dev(pl.ctx, c2_cm.h, C.byref(c2_plan),
                                             C.byref(mode_both), C.byref(c2_ds), c2_iters,
                                             *[ptr(x) for x in c2_out], sh))
        c2_ms = timed(c2_step, max(2, args.steps // 3), 1)
        c2_threads = os.cpu_count() or 1
        c2_sample = min(c2_iters, 2000)
        kind2, times2 = cpu_reference(c2_s, c2_plan, mode_both, c2_sample, 2, 0, c2_threads,
                                      (c2_model, c2_cluster, c2_book), bs=c2_l)
        out["config2"] = {
            "metric": "inter-reordered iterations/s (disaggregated_reorder default mode, LLaVA "
                      "ViT-L + 7B, PP 1/2/1, 32 microbatches/iteration, 10K iterations)",
            "value": c2_iters / (c2_ms / 1e3), "unit": "iterations/s", "ms_per_step": c2_ms,
            "cpu_baseline": {"value": c2_sample / float(np.median(times2)),
                             "unit": "iterations/s", "cores": c2_threads, "kind": kind2,
                             "sample": f"first {c2_sample} iterations"}}
        # exhaustive ordering scorer: every ordering of
        # l = 10 microbatches, p = 4, scored by the 1F1B makespan
        rng_x = np.random.default_rng(10)
        fx, bx = H.skewed_times(rng_x.lognormal(0, 0.5, 10), 4, 0.4)
        pl.exhaustive_order(fx, bx, 1)
        t0 = time.perf_counter()
        for _ in range(3):
            bt_x, _o, _a = pl.exhaustive_order(fx, bx, 1)
        ex_dt = (time.perf_counter() - t0) / 3
        out["exhaustive_orders"] = {"metric": "orderings scored/s (exhaustive 1F1B makespan, "
                                              "l = 10, p = 4; tests/test_reorder.cpp:215-239)",
                                    "value": 3628800 / ex_dt, "unit": "orderings/s",
                                    "ms_per_call": ex_dt * 1e3,
                                    "timing": "host wall clock around the C-ABI call"}
        # trace ingest: write_trace JSONL of a 16M-sample
        # stream -> sample CSR; device-resident bytes, and the host API
        from paper_2408_04275_b200.workload import write_trace
        import torch
        tr_base_n = 1 << 20
        tr_base = write_trace(synth_stream(tr_base_n, seed=7))
        tr_reps = 16
        tr_bytes = tr_base * tr_reps
        tr_n = tr_base_n * tr_reps
        d_tr = torch.frombuffer(bytearray(tr_bytes), dtype=torch.uint8).cuda()
        tr_res = pl.ingest_trace_dev(d_tr.data_ptr(), len(tr_bytes), 8192)
        tr_out = {"text_tokens": torch.empty(tr_n, dtype=torch.int32, device="cuda"),
                  "image_offsets": torch.empty(tr_n + 1, dtype=torch.int32, device="cuda"),
                  "image_tokens": torch.empty(max(1, tr_res.n_image), dtype=torch.int32,
                                              device="cuda"),
                  "audio_offsets": torch.empty(tr_n + 1, dtype=torch.int32, device="cuda"),
                  "audio_tokens": torch.empty(max(1, tr_res.n_audio), dtype=torch.int32,
                                              device="cuda")}
        tr_o = dict(cap_samples=tr_n, cap_image=tr_res.n_image, cap_audio=tr_res.n_audio,
                    **{k: v.data_ptr() for k, v in tr_out.items()})
        for _ in range(2):
            pl.ingest_trace_dev(d_tr.data_ptr(), len(tr_bytes), 8192, tr_o)
        torch.cuda.synchronize()
        tr_ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            pl.ingest_trace_dev(d_tr.data_ptr(), len(tr_bytes), 8192, tr_o)
            torch.cuda.synchronize()
            tr_ts.append(time.perf_counter() - t0)
        tr_dt = float(np.median(tr_ts))
        t0 = time.perf_counter()
        tr_host = pl.ingest_trace(tr_bytes, 8192)
        tr_e2e = time.perf_counter() - t0
        assert tr_host.n == tr_n
        del d_tr, tr_out
        tr_cpu = {}
        try:
            import oracle
            if oracle.ref_available():
                sl = tr_base[: len(tr_base) // 8]
                sl = sl[: sl.rindex(b"\n") + 1]
                t0 = time.perf_counter()
                r_cpu = oracle.ref().ingest_trace(sl, 8192)
                tr_cpu = {"value": r_cpu.n / (time.perf_counter() - t0), "unit": "samples/s",
                          "cores": 1, "kind": "reference",
                          "sample": f"first {r_cpu.n} lines ({len(sl)} bytes); ingest_trace "
                                    "reads one std::istream sequentially"}
        except Exception as ex:  # pragma: no cover
            tr_cpu = {"error": str(ex)}
        out["ingest"] = {"metric": "trace samples ingested/s (ingest_trace, write_trace JSONL "
                                   "of the 16M-sample mixed stream -> sample CSR)",
                         "value": tr_n / tr_dt, "unit": "samples/s", "ms_per_call": tr_dt * 1e3,
                         "bytes": len(tr_bytes), "gb_per_s": len(tr_bytes) / tr_dt / 1e9,
                         "timing": "host wall clock around dtb_ingest_trace_dev (device "
                                   "bytes -> device CSR, includes its internal syncs)",
                         "e2e": {"value": tr_n / tr_e2e, "unit": "samples/s",
                                 "h2d_bytes_per_step": len(tr_bytes),
                                 "d2h_bytes_per_step": 4 * (3 * tr_n + 2 + tr_res.n_image +
                                                            tr_res.n_audio),
                                 "path": "dtb_ingest_trace (pageable host bytes -> host CSR)"},
                         "cpu_baseline": tr_cpu}
        # orchestration search, BASELINE config 3
        smodel, scluster, sbook, sbs, sstats = search_workload()
        scm = pl.cost_model(smodel, scluster, sbook)
        res = A.OrchestrationResult()
        for _ in range(2):
            pl._check(lib.model_orchestration(pl.ctx, scm.h, C.byref(sstats), sbs, 1,
                                              C.byref(res), None, 0))
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            pl._check(lib.model_orchestration(pl.ctx, scm.h, C.byref(sstats), sbs, 1,
                                              C.byref(res), None, 0))
        s_dt = (time.perf_counter() - t0) / reps
        out["search"] = {"metric": "orchestration candidates/s (model_orchestration, 72B MLLM, "
                                   "1172 GPUs, BS 1920)",
                         "value": res.candidates_evaluated / s_dt, "unit": "candidates/s",
                         "ms_per_search": s_dt * 1e3, "candidates": res.candidates_evaluated,
                         "timing": "host wall clock around the C-ABI call (includes "
                                   "enumeration, solve, reduce, D2H)"}
        # FP64 roofline of the search: the device part of the same search
        # (dtb_orchestration_shard_dev, one shard) timed with CUDA events on
        # its stream; FP64 instructions per search from the committed ncu
        # count (profiles/r02_fp64_ops.json)
        try:
            fops = json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_ops.json")))
            kinst = fops["search_config3"]["kernels"]
            inst = sum(k["dadd"] + k["dmul"] + k["dfma"] for k in kinst.values())
            rec = torch.zeros(C.sizeof(A.Candidate), dtype=torch.uint8, device="cuda")
            evc = torch.zeros(1, dtype=torch.int64, device="cuda")
            st_s = torch.cuda.Stream()
            call = lambda: pl._check(lib.orchestration_shard_dev(
                pl.ctx, scm.h, C.byref(sstats), sbs, 1, 0, 1, C.c_void_p(rec.data_ptr()),
                C.c_void_p(evc.data_ptr()), C.c_void_p(st_s.cuda_stream)))
            for _ in range(2):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st_s)
            for _ in range(reps):
                call()
            e1.record(st_s)
            torch.cuda.synchronize()
            dev_s = e0.elapsed_time(e1) / 1e3 / reps
            ach = inst / dev_s
            out["search"]["roofline"] = {
                "bound": "fp64", "kernel": "orch_kernel (+ enumeration, screen, reduce kernels "
                "of dtb_orchestration_shard_dev)", "achieved": ach,
                "peak": fops["peak_fp64_instr_per_s"], "unit": "FP64 instr/s",
                "frac": ach / fops["peak_fp64_instr_per_s"], "fp64_instr_per_search": inst,
                "ms_per_search_device": dev_s * 1e3, "peak_source": fops["peak_source"],
                "counts_source": fops["search_config3"]["source"]}
        except Exception as ex:  # counts file absent: no FP64 block
            out["search"]["roofline"] = {"unavailable": str(ex)[:120]}
        # BASELINE config 5: search at BS 16,384, then reorder the resident
        # 16M stream with the CHOSEN plan (ReorderMode{intra})
        from paper_2408_04275_b200.api import PlanSpec
        c5 = A.OrchestrationResult()
        c5_search = []
        for it in range(3):
            t0 = time.perf_counter()
            pl._check(lib.model_orchestration(pl.ctx, scm.h, C.byref(sstats), BS, 1,
                                              C.byref(c5), None, 0))
            c5_search.append(time.perf_counter() - t0)
        c5_plan = PlanSpec.from_c(c5.best)
        c5_pc = c5.best
        c5_dp = c5_pc.unit[1].dp
        c5_o = [torch.empty(my_batches * c5_dp, dtype=torch.float64, device="cuda")
                for _ in range(2)] + [torch.empty(my_batches, dtype=torch.float64,
                                                  device="cuda") for _ in range(2)]

        def c5_step():
            pl._check(lib.reorder_stream_dev(pl.ctx, scm.h, C.byref(c5_pc), C.byref(mode_intra),
                                             C.byref(ds), my_batches, ptr(out_order),
                                             *[ptr(x) for x in c5_o], ptr(kept), sh))
        c5_ms = timed(c5_step, max(2, args.steps // 3), 1)
        c5_s = float(np.median(c5_search))
        out["config5"] = {
            "metric": "search + reorder of the 16M stream with the chosen plan (model_orchestration "
                      "72B MLLM, 1172 GPUs, BS 16384; disaggregated_reorder ReorderMode{intra})",
            "plan": repr(c5_plan), "search_ms": c5_s * 1e3, "reorder_ms": c5_ms,
            "value": my_batches * BS / (c5_s + c5_ms / 1e3), "unit": "samples/s",
            "candidates": c5.candidates_evaluated,
            "timing": "search: host wall clock around the C-ABI call; reorder: CUDA events"}
        # CPU baseline: the compiled reference on this host's cores
        threads = os.cpu_count() or 1
        sample_batches = max(1, min(my_batches, 2 * threads))
        kind, times = cpu_reference(samples, plan_c, mode_intra, sample_batches, 2, 0, threads,
                                    (model, cluster, book))
        t = float(np.median(times))
        kind1, times1 = cpu_reference(samples, plan_c, mode_intra, 4, 2, 0, 1,
                                      (model, cluster, book))
        out["cpu_baseline"] = {"value": sample_batches * BS / t, "unit": "samples/s",
                               "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                               "sample": f"first {sample_batches} global batches of the stream "
                                         f"(x{BS} samples), std::thread fan-out over batches",
                               "single_thread": {"value": 4 * BS / float(np.median(times1)),
                                                 "unit": "samples/s", "cores": 1,
                                                 "sample": "first 4 global batches, one thread"}}
        try:
            kind_s, th_s, cps, s_cpu, _ = cpu_search(threads)
            out["search"]["cpu_baseline"] = {"value": cps, "unit": "candidates/s",
                                             "cores": th_s, "kind": kind_s,
                                             "seconds": s_cpu}
        except Exception as ex:  # pragma: no cover
            out["search"]["cpu_baseline"] = {"error": str(ex)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
