"""Multi-GPU check of dtb_reorder_stream_shard_dev (run under torchrun, one
process per GPU): every rank reorders its batch range of ONE stream and the
library exchanges the ordering over NVLink into every rank's replica.  Also
the search sharded over the ranks (dtb_orchestration_shard_dev), the winners
all-gathered and folded by dtb_best_reduce_dev, against model_orchestration.  Each
rank checks the whole replica against a single-GPU reorder of the whole
stream (dtb_reorder_stream_dev on its own GPU) and its per-batch outputs at
its own batch positions; then times the sharded step (CUDA events, max over
ranks) against the single-GPU step.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/peer_check.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import helpers as H
    from paper_2408_04275_b200 import _capi as A
    from paper_2408_04275_b200 import native
    from paper_2408_04275_b200.workload import synth_stream

    bs, dp = 16384, 128
    n_batches = int(os.environ.get("PEER_BATCHES", "1024"))
    pl = native.planner(local)
    lib = pl.lib
    cm = pl.cost_model(H.desk_model(), H.desk_cluster(1172), H.desk_book())
    plan = H.plan((1, dp, 1), (1, dp, 2), (1, dp, 1), bs).to_c()
    results = {}
    for fam in ("mixed", "dense"):
        for inter in (0, 1):
            nb = n_batches if not inter else min(n_batches, 64)
            s = synth_stream(nb * bs, seed=1000, family=fam)
            total = s.n
            dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
            d = [dev(s.image_offsets), dev(s.image_tokens), dev(s.audio_offsets), dev(s.audio_tokens)]
            ds = A.Samples(total, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in d])
            mode = A.ReorderMode(1, inter, 0)
            f64 = lambda k: torch.zeros(k, dtype=torch.float64, device="cuda")
            full = [torch.empty(total, dtype=torch.int32, device="cuda"), f64(nb * dp), f64(nb * dp),
                    f64(nb), f64(nb), torch.empty(nb, dtype=torch.uint8, device="cuda")]
            ptr = lambda t: C.c_void_p(t.data_ptr())
            stream = torch.cuda.Stream()
            sh = C.c_void_p(stream.cuda_stream)
            one = lambda: pl._check(lib.reorder_stream_dev(pl.ctx, cm.h, C.byref(plan), C.byref(mode),
                                                           C.byref(ds), nb, *[ptr(x) for x in full], sh))
            replica, handle = pl.peer_buffer_create(total)
            handles = [None] * world
            dist.all_gather_object(handles, handle)
            group = pl.peer_group_open(rank, world, replica, total, handles)
            mine = [f64(nb * dp), f64(nb * dp), f64(nb), f64(nb),
                    torch.zeros(nb, dtype=torch.uint8, device="cuda")]
            shard = lambda: pl._check(lib.reorder_stream_shard_dev(
                pl.ctx, cm.h, C.byref(plan), C.byref(mode), C.byref(ds), nb, group,
                *[ptr(x) for x in mine], sh))
            with torch.cuda.stream(stream):
                one()
                shard()
            torch.cuda.synchronize()
            dist.barrier()
            rep_host = np.empty(total, dtype=np.uint16)
            import ctypes.util
            rt = C.CDLL(ctypes.util.find_library("cudart") or "libcudart.so")
            rt.cudaMemcpy(C.c_void_p(rep_host.ctypes.data), C.c_void_p(replica),
                          C.c_size_t(2 * total), 2)  # cudaMemcpyDeviceToHost
            want = full[0].cpu().numpy()
            first, count = pl.shard_range(nb, rank, world)
            ok_order = bool(np.array_equal(rep_host.astype(np.int32), want))
            sl = slice(first, first + count)
            ok_t = bool(np.array_equal(mine[2].cpu().numpy()[sl], full[3].cpu().numpy()[sl]) and
                        np.array_equal(mine[3].cpu().numpy()[sl], full[4].cpu().numpy()[sl]))
            ok_l = bool(np.array_equal(mine[0].cpu().numpy().reshape(nb, dp)[sl],
                                       full[1].cpu().numpy().reshape(nb, dp)[sl]))

            def timed(fn, steps=10, warm=3):
                for _ in range(warm):
                    fn()
                torch.cuda.synchronize()
                dist.barrier()
                evs = []
                for _ in range(steps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    evs.append((e0, e1))
                torch.cuda.synchronize()
                t = torch.tensor([float(np.mean([a.elapsed_time(b) for a, b in evs]))], device="cuda",
                                 dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                return float(t.item())
            g = C.c_void_p()
            pl._check(lib.reorder_stream_graph_create(pl.ctx, cm.h, C.byref(plan), C.byref(mode),
                                                      C.byref(ds), nb, group, None,
                                                      *[ptr(x) for x in mine], C.byref(g)))
            # this rank's batch range alone on this GPU (no exchange)
            first, count = pl.shard_range(nb, rank, world)
            # (offsets are absolute into the whole CSR: only the offset arrays move)
            dsh = A.Samples(count * bs, None,
                            C.cast(d[0].data_ptr() + 4 * first * bs, C.POINTER(C.c_int32)),
                            C.cast(d[1].data_ptr(), C.POINTER(C.c_int32)),
                            C.cast(d[2].data_ptr() + 4 * first * bs, C.POINTER(C.c_int32)),
                            C.cast(d[3].data_ptr(), C.POINTER(C.c_int32)))
            half = [torch.empty(count * bs, dtype=torch.int32, device="cuda"), f64(count * dp),
                    f64(count * dp), f64(count), f64(count), torch.empty(count, dtype=torch.uint8, device="cuda")]
            local = lambda: pl._check(lib.reorder_stream_dev(pl.ctx, cm.h, C.byref(plan), C.byref(mode),
                                                             C.byref(dsh), count, *[ptr(x) for x in half], sh))
            with torch.cuda.stream(stream):
                t_one = timed(one)
                t_local = timed(local)
                t_shard = timed(shard)
                t_graph = timed(lambda: pl._check(lib.graph_launch(g, sh)))
            pl._check(lib.graph_destroy(g))
            res = torch.tensor([ok_order and ok_t and ok_l], dtype=torch.int32, device="cuda")
            dist.all_reduce(res, op=dist.ReduceOp.MIN)
            results[f"{fam} inter={inter}"] = {
                "batches": nb, "all_ranks_bit_exact": bool(res.item()), "ms_single_gpu": t_one,
                "ms_own_range_no_exchange": t_local,
                "ms_sharded_with_exchange": t_shard, "speedup": t_one / t_shard,
                "ms_sharded_graph": t_graph, "speedup_graph": t_one / t_graph}
            pl.peer_group_close(group)
            dist.barrier()
            pl.peer_buffer_destroy(replica)
    # the search sharded over the ranks (dtb_orchestration_shard_dev), the
    # winners all-gathered and folded on the device (dtb_best_reduce_dev)
    from paper_2408_04275_b200.api import PlanSpec, stats_to_c
    m72, cl72, bk72 = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
    st72 = stats_to_c(m72.seq_len, 2048.0, 2048.0)
    cm72 = pl.cost_model(m72, cl72, bk72)
    want = pl.model_orchestration(cm72, st72, 1920)
    csz = C.sizeof(A.Candidate)
    rec = torch.zeros(csz, dtype=torch.uint8, device="cuda")
    evn = torch.zeros(1, dtype=torch.int64, device="cuda")
    sh0 = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    pl._check(lib.orchestration_shard_dev(pl.ctx, cm72.h, C.byref(st72), 1920, 1, rank, world,
                                          C.c_void_p(rec.data_ptr()), C.c_void_p(evn.data_ptr()), sh0))
    recs = torch.zeros(world * csz, dtype=torch.uint8, device="cuda")
    evs = torch.zeros(world, dtype=torch.int64, device="cuda")
    dist.all_gather_into_tensor(recs, rec)
    dist.all_gather_into_tensor(evs, evn)
    best = torch.zeros(csz, dtype=torch.uint8, device="cuda")
    pl._check(lib.best_reduce_dev(pl.ctx, C.c_void_p(recs.data_ptr()), world, C.c_void_p(best.data_ptr()), sh0))
    torch.cuda.synchronize()
    c = A.Candidate.from_buffer_copy(best.cpu().numpy().tobytes())
    ok_search = bool(c.feasible == 1 and PlanSpec.from_c(c.plan) == want["best"] and
                     (c.times.t_warm, c.times.t_steady, c.times.t_iter) == want["times"] and
                     int(evs.sum().item()) == want["candidates_evaluated"])
    res = torch.tensor([1 if ok_search else 0], dtype=torch.int32, device="cuda")
    dist.all_reduce(res, op=dist.ReduceOp.MIN)
    results["search sharded"] = {"all_ranks_bit_exact": bool(res.item()),
                                 "candidates": int(evs.sum().item())}
    if rank == 0:
        print(json.dumps({"world": world, "results": results}, indent=1), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
