"""N > 1 host logic on CPU: world_size-2 `gloo` process groups.

Each rank reorders its global-batch range (shard.batch_range) and searches
its tuple shard (shard.tuple_shard); results are exchanged with gloo
collectives and must equal the single-rank computation — the same sharding
bench.py runs over NCCL with one process per GPU.  The planner here is the
CPU oracle (this container has no GPU); the sharding/folding code under test
is the product's host code (paper_2408_04275_b200/shard.py)."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import helpers as H
    import oracle
    from paper_2408_04275_b200 import shard
    from paper_2408_04275_b200.api import stats_to_c
    from paper_2408_04275_b200.workload import synth_stream

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pl = oracle.port()
    model, cluster, book = H.desk_model(), H.desk_cluster(64), H.desk_book()
    cm = pl.cost_model(model, cluster, book)
    # ---- reorder stream, batch-range sharding, all-gather of the orders
    bs, n_batches = 256, 7
    plan = H.plan((1, 8, 1), (1, 8, 2), (1, 8, 1), bs)
    stream = synth_stream(n_batches * bs, 99, "mixed")
    first, count = shard.batch_range(n_batches, rank, world)
    mine = pl.reorder_stream(cm, plan, stream.slice(first * bs, (first + count) * bs), count,
                             inter=True)
    parts = [None] * world
    dist.all_gather_object(parts, {k: np.asarray(v) for k, v in mine.items()})
    # ---- orchestration, strided tuple shards, winner fold
    stats = stats_to_c(model.seq_len, 1000.0, 1000.0)
    full = pl.model_orchestration(cm, stats, 64, keep_candidates=True)
    cands = full["candidates"]
    local = shard.fold_winners(cands[i] for i in shard.tuple_shard(len(cands), rank, world))
    winners = [None] * world
    dist.all_gather_object(winners, local)
    if rank == 0:
        whole = pl.reorder_stream(cm, plan, stream, n_batches, inter=True)
        for k, v in whole.items():
            got = np.concatenate([p[k] for p in parts])
            assert np.array_equal(got, np.asarray(v)), k
        best = shard.fold_winners(winners)
        assert best.plan == full["best"], (best.plan, full["best"])
        assert best.times == full["times"]
        open(os.path.join(out_dir, "ok"), "w").write("ok")
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_rank(tmp_path, port):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok").exists()


def test_batch_range_covers_the_stream():
    from paper_2408_04275_b200 import shard
    for n in (1, 7, 1024):
        for w in (1, 2, 3, 8):
            spans = [shard.batch_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == n
            assert all(a + c == b for (a, c), (b, _) in zip(spans, spans[1:]))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
