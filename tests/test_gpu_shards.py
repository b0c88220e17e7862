"""Multi-GPU entry points of the product on the GPU.

* dtb_orchestration_shard_dev + dtb_best_reduce_dev: the BASELINE config 3
  search split into 2, 3 and 4 shards (run here one after another on one GPU:
  the shard arithmetic is what multi-GPU runs distribute) and folded on the
  device must give model_orchestration's winner and candidate count, i.e.
  the reference's (src/orchestrator.cpp:380-405, tie-break :211-233).
* dtb_reorder_stream_shard_dev over a one-rank peer group equals
  dtb_reorder_stream_dev; the replica holds the ordering as u16.
* With two or more GPUs visible: tools/peer_check.py under torchrun (two
  ranks, NCCL for the handle exchange only) — every rank's replica and outputs
  bit-exact against a single-GPU reorder of the whole stream, and the search
  sharded over the two ranks, folded on the device, equal to
  model_orchestration's winner.
"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import helpers as H
from paper_2408_04275_b200 import _capi as A
from paper_2408_04275_b200.api import stats_to_c

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("shards", [2, 3, 4])
def test_search_shards_fold(gpu, shards):
    import torch
    m, cl, bk = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
    st = stats_to_c(m.seq_len, 2048.0, 2048.0)
    cm = gpu.cost_model(m, cl, bk)
    want = gpu.model_orchestration(cm, st, 1920)
    rec = torch.zeros(shards * C.sizeof(A.Candidate), dtype=torch.uint8, device="cuda")
    ev = torch.zeros(shards, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    sh = C.c_void_p(stream.cuda_stream)
    for i in range(shards):
        gpu._check(gpu.lib.orchestration_shard_dev(
            gpu.ctx, cm.h, C.byref(st), 1920, 1, i, shards,
            C.c_void_p(rec.data_ptr() + i * C.sizeof(A.Candidate)),
            C.c_void_p(ev.data_ptr() + 8 * i), sh))
    best = torch.zeros(C.sizeof(A.Candidate), dtype=torch.uint8, device="cuda")
    gpu._check(gpu.lib.best_reduce_dev(gpu.ctx, C.c_void_p(rec.data_ptr()), shards,
                                       C.c_void_p(best.data_ptr()), sh))
    torch.cuda.synchronize()
    raw = best.cpu().numpy().tobytes()
    c = A.Candidate.from_buffer_copy(raw)
    assert c.feasible == 1
    from paper_2408_04275_b200.api import PlanSpec
    assert PlanSpec.from_c(c.plan) == want["best"]
    assert (c.times.t_warm, c.times.t_steady, c.times.t_iter) == want["times"]
    assert int(ev.sum().item()) == want["candidates_evaluated"] == 140370


def test_stream_shard_one_rank(gpu):
    import torch
    from paper_2408_04275_b200.workload import synth_stream
    bs, dp, nb = 16384, 128, 24
    s = synth_stream(nb * bs, seed=77, family="mixed")
    cm = gpu.cost_model(H.desk_model(), H.desk_cluster(1172), H.desk_book())
    plan = H.plan((1, dp, 1), (1, dp, 2), (1, dp, 1), bs).to_c()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d = [dev(s.image_offsets), dev(s.image_tokens), dev(s.audio_offsets), dev(s.audio_tokens)]
    ds = A.Samples(s.n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in d])
    f64 = lambda k: torch.zeros(k, dtype=torch.float64, device="cuda")
    ptr = lambda t: C.c_void_p(t.data_ptr())
    sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for inter in (0, 1):
        mode = A.ReorderMode(1, inter, 0)
        full = [torch.empty(s.n, dtype=torch.int32, device="cuda"), f64(nb * dp), f64(nb * dp),
                f64(nb), f64(nb), torch.zeros(nb, dtype=torch.uint8, device="cuda")]
        gpu._check(gpu.lib.reorder_stream_dev(gpu.ctx, cm.h, C.byref(plan), C.byref(mode),
                                              C.byref(ds), nb, *[ptr(x) for x in full], sh))
        replica, handle = gpu.peer_buffer_create(s.n)
        group = gpu.peer_group_open(0, 1, replica, s.n, [handle])
        mine = [f64(nb * dp), f64(nb * dp), f64(nb), f64(nb),
                torch.zeros(nb, dtype=torch.uint8, device="cuda")]
        gpu._check(gpu.lib.reorder_stream_shard_dev(gpu.ctx, cm.h, C.byref(plan), C.byref(mode),
                                                    C.byref(ds), nb, group,
                                                    *[ptr(x) for x in mine], sh))
        torch.cuda.synchronize()
        import ctypes.util
        rt = C.CDLL(ctypes.util.find_library("cudart") or "libcudart.so")
        host = np.empty(s.n, dtype=np.uint16)
        assert rt.cudaMemcpy(C.c_void_p(host.ctypes.data), C.c_void_p(replica),
                             C.c_size_t(2 * s.n), 2) == 0
        np.testing.assert_array_equal(host.astype(np.int32), full[0].cpu().numpy())
        for a, b in zip(mine, full[1:]):
            np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
        gpu.peer_group_close(group)
        gpu.peer_buffer_destroy(replica)


def test_peer_exchange_two_gpus():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU visible: the two-rank exchange runs in tools/peer_check.py "
                    "(profiles/r02_peer_check_n2.json)")
    env = dict(os.environ, PEER_BATCHES="64")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", os.path.join(ROOT, "tools", "peer_check.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout[r.stdout.index("{"):]
    res = json.loads(out)["results"]
    assert res and all(v["all_ranks_bit_exact"] for v in res.values()), res
