"""Seeded inputs of the golden fixtures (tests/golden/*.npz) and the calls
that produce their outputs on any planner backend.  make_golden.py records
the compiled reference's outputs; tests/test_golden_fixtures.py replays the
same calls on the oracle port (CPU) and the CUDA path (GPU) and compares
bit-exactly."""
from __future__ import annotations

import numpy as np

from paper_2408_04275_b200.api import DESCENDING, stats_to_c
from paper_2408_04275_b200.workload import synth_stream

import helpers as H


def stream_c1(pl):
    """BASELINE config 1 shape (512 samples, DP 8) x 6 batches, default mode
    and intra-only, plus one descending batch set."""
    cm = pl.cost_model(H.desk_model(), H.desk_cluster(64), H.desk_book())
    plan = H.plan((1, 8, 1), (1, 8, 2), (1, 8, 1), 512)
    s = synth_stream(6 * 512, 20261018, "mixed")
    a = pl.reorder_stream(cm, plan, s, 6, inter=True)
    b = pl.reorder_stream(cm, plan, s, 6, inter=False)
    c = pl.reorder_stream(cm, plan, s.slice(0, 1024), 2, inter=True, sort_order=DESCENDING)
    out = {}
    for tag, r in (("both", a), ("intra", b), ("desc", c)):
        for k, v in r.items():
            out[f"{tag}_{k}"] = np.asarray(v)
    return out


def stream_c4_batch(pl):
    """One BASELINE config 4 global batch (16384 samples, DP 128), intra."""
    cm = pl.cost_model(H.desk_model(), H.desk_cluster(1172), H.desk_book())
    plan = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384)
    s = synth_stream(16384, 42, "mixed")
    r = pl.reorder_stream(cm, plan, s, 1, inter=False)
    return {k: np.asarray(v) for k, v in r.items()}


def inter_c2(pl):
    """BASELINE config 2 shape: 64 LLaVA iterations of 32 microbatches,
    default mode."""
    cm = pl.cost_model(H.llava_model(), H.a800_cluster(64), H.llava_book())
    plan = H.plan((1, 1, 1), (1, 1, 2), (1, 1, 1), 32)
    s = synth_stream(64 * 32, 7, "skewed")
    r = pl.reorder_stream(cm, plan, s, 64, inter=True)
    return {k: np.asarray(v) for k, v in r.items()}


def search_small(pl):
    """model_orchestration on the desk model (64 GPUs) and the 72B model on
    112 GPUs; brute_force_oracle and rigid_baseline on 32 GPUs."""
    out = {}
    for tag, model, cluster, book, bs in (
            ("desk", H.desk_model(), H.desk_cluster(64), H.desk_book(), 64),
            ("mllm", H.mllm72b_model(), H.a800_cluster(112), H.mllm72b_book(), 240)):
        cm = pl.cost_model(model, cluster, book)
        r = pl.model_orchestration(cm, stats_to_c(model.seq_len, 1000.0, 1000.0), bs)
        out[f"{tag}_plan"] = np.asarray(plan_vec(r["best"]))
        out[f"{tag}_times"] = np.asarray(r["times"])
        out[f"{tag}_evaluated"] = np.asarray(r["candidates_evaluated"])
    model, cluster, book = H.desk_model(), H.desk_cluster(32), H.desk_book()
    cm = pl.cost_model(model, cluster, book)
    st = stats_to_c(model.seq_len, 1000.0, 1000.0)
    r = pl.brute_force_oracle(cm, st, 64)
    out["brute_plan"] = np.asarray(plan_vec(r["best"]))
    out["brute_times"] = np.asarray(r["times"])
    out["brute_evaluated"] = np.asarray(r["candidates_evaluated"])
    out["rigid_plan"] = np.asarray(plan_vec(pl.rigid_baseline(cm, st, 64)))
    return out


def exhaustive(pl):
    rng = np.random.default_rng(99)
    f, b = H.skewed_times(rng.lognormal(0, 0.5, 7), 3, 0.4)
    t, order, allt = pl.exhaustive_order(f, b, 1, with_all=True)
    return {"best_time": np.asarray(t), "order": np.asarray(order), "all": allt}


def plan_vec(p):
    return [p.encoder.tp, p.encoder.dp, p.encoder.pp, p.backbone.tp, p.backbone.dp,
            p.backbone.pp, p.generator.tp, p.generator.dp, p.generator.pp, p.global_batch, p.vpp]


CASES = {"stream_c1": stream_c1, "stream_c4_batch": stream_c4_batch, "inter_c2": inter_c2,
         "search_small": search_small, "exhaustive": exhaustive}
