"""Benchmark: DistTrain reorder hot path on B200 (BASELINE.json config 4).

Workload: a 16,777,216-sample synthetic image+audio stream (variable
resolution -> patch tokens, audio clips) in global batches of 16,384, plan
DP_lm = DP_me = DP_mg = 128, PP 1/2/1 (l = 128 microbatches per pipeline), the
reference's desk-shaped cost profile.  One step = `disaggregated_reorder`
(src/reorder.cpp:319-396) over every global batch of the stream with
ReorderMode{intra=true, inter=false}: per-sample cost, stable sort, greedy
equal-count partition, keep-if-no-worse, group loads and both simulated
iteration times — the sort/partition path the north_star's HBM target names.
The full default mode (intra + inter) and the orchestration search
(config 3) are measured too and reported under "modes".

N GPUs (torchrun): the stream is split by global-batch range (strong
scaling, fixed 16M total); no collective on the data path.  `value` = all
samples / max-over-ranks device time.

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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=STREAM)
    ap.add_argument("--no-extras", action="store_true", help="skip modes/e2e/cpu legs")
    return ap.parse_args()


def dist_init(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
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


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, idx):
        self.idx = idx
        self.proc = None
        self.path = f"/tmp/dtb_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_reference(samples, plan_c, mode, n_batches, steps, warmup, threads, cm):
    """Reference CPU path (all host threads) on n_batches global batches."""
    import oracle
    from paper_2408_04275_b200 import _capi as A
    pl, kind = oracle.best()
    lib = pl.lib
    if not lib.has("stream_prepare"):
        raise RuntimeError("oracle lacks stream entry points")
    sub = samples.slice(0, n_batches * BS)
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


def main():
    args = parse()
    rank, world, local = dist_init(args.gpus)
    model, cluster, book, plan = workload()
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200.workload import synth_stream

    n_batches_total = args.samples // BS
    my_batches = n_batches_total // world + (1 if rank < n_batches_total % world else 0)
    first_batch = rank * (n_batches_total // world) + min(rank, n_batches_total % world)
    plan_c = plan.to_c()
    mode_intra = A.ReorderMode(1, 0, 0)
    mode_both = A.ReorderMode(1, 1, 0)

    if args.impl == "reference":
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        sample_batches = max(1, min(n_batches_total, 4 * threads))
        samples = synth_stream(sample_batches * BS, seed=1, family="mixed")
        kind, times = cpu_reference(samples, plan_c, mode_intra, sample_batches, args.steps,
                                    args.warmup, threads, (model, cluster, book))
        t = float(np.median(times))
        v = sample_batches * BS / t
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
               "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "int32/int64 keys, f64 costs",
               "data": "synthetic (PCG64 mixed image+audio stream)",
               "config": {"workload": "BASELINE config 4 (bounded CPU sample)",
                          "global_batch": BS, "dp": DP, "pp": "1/2/1",
                          "mode": "intra", "sample_batches": sample_batches},
               "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads,
                                "kind": kind,
                                "sample": f"{sample_batches} global batches x {BS}"},
               "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    import torch
    torch.cuda.set_device(local)
    from paper_2408_04275_b200 import native
    pl = native.planner(local)
    lib = pl.lib
    cm = pl.cost_model(model, cluster, book)

    samples = synth_stream(my_batches * BS, seed=1000 + first_batch, family="mixed")
    n = samples.n
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_io, d_it = dev(samples.image_offsets), dev(samples.image_tokens)
    d_ao, d_at = dev(samples.audio_offsets), dev(samples.audio_tokens)
    ds = A.Samples(n, None, C.cast(d_io.data_ptr(), C.POINTER(C.c_int32)),
                   C.cast(d_it.data_ptr(), C.POINTER(C.c_int32)),
                   C.cast(d_ao.data_ptr(), C.POINTER(C.c_int32)),
                   C.cast(d_at.data_ptr(), C.POINTER(C.c_int32)))
    out_order = torch.empty(n, dtype=torch.int32, device="cuda")
    lb = torch.empty(my_batches * DP, dtype=torch.float64, device="cuda")
    la = torch.empty_like(lb)
    tb = torch.empty(my_batches, dtype=torch.float64, device="cuda")
    ta = torch.empty_like(tb)
    kept = torch.empty(my_batches, dtype=torch.uint8, device="cuda")
    # L2 flush buffer (inputs are > L2 anyway at full size; flush keeps it honest)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    sh = C.c_void_p(stream.cuda_stream)

    def step(mode):
        pl._check(lib.reorder_stream_dev(pl.ctx, cm.h, C.byref(plan_c), C.byref(mode), C.byref(ds),
                                         my_batches, C.c_void_p(out_order.data_ptr()),
                                         C.c_void_p(lb.data_ptr()), C.c_void_p(la.data_ptr()),
                                         C.c_void_p(tb.data_ptr()), C.c_void_p(ta.data_ptr()),
                                         C.c_void_p(kept.data_ptr()), sh))

    def k1():
        pl._check(lib.intra_stream_dev(pl.ctx, BS, DP, 0, C.byref(ds), my_batches,
                                       C.c_void_p(out_order.data_ptr()), C.c_void_p(lb.data_ptr()),
                                       C.c_void_p(la.data_ptr()), C.c_void_p(kept.data_ptr()), sh))

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
        ms = [s.elapsed_time(e) for s, e in evs]
        return float(np.mean(ms)), ms

    with Clocks(local) as clk:
        ms_local, _ = timed(lambda: step(mode_intra), args.steps, args.warmup)
    ms = max_over_ranks(ms_local, world)
    total = n_batches_total * BS
    value = total / (ms / 1e3)
    out = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "int32 tokens / int64 loads / f64 stage times",
           "data": "synthetic (PCG64 mixed image+audio stream, random-free desk cost profile)",
           "config": {"workload": "BASELINE config 4: 16M-sample stream, global batch 16384, "
                                  "DP 128, PP 1/2/1, ReorderMode{intra}",
                      "samples": total, "global_batch": BS, "dp": DP,
                      "parallelism": f"batch-range sharding over {world} GPU(s)",
                      "l2": "256 MiB flush written between timed steps; inputs > L2"},
           "gpu_launches": 8 * 1}
    clocks = clk.summary()
    if clocks:
        out["clocks"] = clocks

    # ---- dominant kernel (sort/partition) roofline
    k1_ms_local, _ = timed(k1, args.steps, args.warmup)
    k1_ms = max_over_ranks(k1_ms_local, world)
    n_img, n_aud = len(samples.image_tokens), len(samples.audio_tokens)
    algo_bytes = (4 * 2 * (n + my_batches) + 4 * (n_img + n_aud)  # offsets + tokens
                  + 4 * n + 2 * 8 * DP * my_batches + my_batches)  # order + loads + kept
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = algo_bytes / (k1_ms_local / 1e3) / 1e9
    out["roofline"] = {"bound": "hbm", "kernel": "intra_fused_kernel", "achieved": achieved,
                       "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                       "algorithmic_bytes_per_launch": algo_bytes,
                       "ms_per_launch": k1_ms_local,
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}

    if not args.no_extras and rank == 0:
        # full default mode (intra + inter)
        both_ms, _ = timed(lambda: step(mode_both), max(2, args.steps // 3), 1)
        out["modes"] = {"intra+inter": {"ms_per_step": both_ms,
                                        "value": my_batches * BS / (both_ms / 1e3)}}
    out["gpu_launches"] = 8
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
