"""BASELINE.json configurations at FULL size, CUDA path vs the compiled
reference (oracle/_ref; the C restatement when absent), bit-exact.

  C2  LLaVA ViT-L + 7B, PP 1/2/1, 32 microbatches per iteration, all 10,000
      iterations in default mode (intra + inter).
  C3  72B MLLM orchestration search for 1,172 GPUs at BS 1,920: best plan,
      times, candidates_evaluated, plus 2,048 sampled solve_subproblem records.
  C4  the 16M-sample mixed stream (1,024 global batches of 16,384, DP 128):
      every batch in ReorderMode{intra}; 32 batches in default mode
      (l = 128 per coupled group); 64 batches with the descending order.
  C5  the C3 model searched at BS 16,384, then one global batch reordered in
      default mode with the CHOSEN plan (DP 16, PP 1/71/7: l = 1,024, p = 79).

The reference runs on all host threads (each batch / problem is one
untouched reference call, `set_threads` in oracle/refshim/ref_capi.cpp).
"""
import os

import numpy as np
import pytest

import helpers as H
from parity_cases import assert_same
from paper_2408_04275_b200.api import DESCENDING, stats_to_c
from paper_2408_04275_b200.workload import synth_stream

pytestmark = pytest.mark.gpu

KEYS = ("output_order", "load_before", "load_after", "t_iter_before", "t_iter_after")


@pytest.fixture(scope="module")
def ora(oracle_best):
    if oracle_best.lib.has("set_threads"):
        oracle_best.lib.set_threads(os.cpu_count() or 1)
    yield oracle_best
    if oracle_best.lib.has("set_threads"):
        oracle_best.lib.set_threads(1)


@pytest.fixture(scope="module")
def c4_stream():
    return synth_stream(1 << 24, seed=1000, family="mixed")


def _desk(gpu, ora, n_gpus=1172):
    model, cluster, book = H.desk_model(), H.desk_cluster(n_gpus), H.desk_book()
    return gpu.cost_model(model, cluster, book), ora.cost_model(model, cluster, book)


def _compare(ra, rb, tag):
    for k in KEYS:
        assert_same(ra[k], rb[k], f"{tag} {k}")


def test_c4_full_stream_intra(gpu, ora, c4_stream):
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384)
    ra = gpu.reorder_stream(ci, pl, c4_stream, 1024, inter=False)
    rb = ora.reorder_stream(co, pl, c4_stream, 1024, inter=False)
    _compare(ra, rb, "C4 intra, 1024 batches")


@pytest.mark.parametrize("bs,dp,nb,fam", [(2048, 16, 301, "mixed"), (2056, 16, 240, "dense"),
                                          (16384, 128, 160, "mixed")])
def test_descending_many_batches(gpu, ora, bs, dp, nb, fam):
    """More listed batches than CTA pairs: the partition kernel's
    single-CTA mode, which in descending order runs two batches per CTA
    with their one-warp greedies side by side (odd counts, n % m != 0)."""
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, dp, 1), (1, dp, 2), (1, dp, 1), bs)
    s = synth_stream(nb * bs, seed=4242 + bs, family=fam)
    ra = gpu.reorder_stream(ci, pl, s, nb, inter=False, sort_order=DESCENDING)
    rb = ora.reorder_stream(co, pl, s, nb, inter=False, sort_order=DESCENDING)
    _compare(ra, rb, f"descending {nb} x {bs} {fam}")


def test_c4_descending(gpu, ora, c4_stream):
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384)
    sub = c4_stream.slice(0, 64 * 16384)
    ra = gpu.reorder_stream(ci, pl, sub, 64, inter=False, sort_order=DESCENDING)
    rb = ora.reorder_stream(co, pl, sub, 64, inter=False, sort_order=DESCENDING)
    _compare(ra, rb, "C4 intra descending, 64 batches")


@pytest.mark.parametrize("order", [0, 1])
def test_c4_shape_dense_kept(gpu, ora, order):
    """The dense family (every sample has an image) at the C4 batch shape:
    the greedy split is kept on most batches, so the stable counting scatter
    (and, descending, the general rounds) run on every batch."""
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384)
    s = synth_stream(48 * 16384, seed=77, family="dense")
    ra = gpu.reorder_stream(ci, pl, s, 48, inter=False, sort_order=order, with_kept=True)
    rb = ora.reorder_stream(co, pl, s, 48, inter=False, sort_order=order)
    _compare(ra, rb, f"C4 shape dense order {order}")
    assert ra["greedy_kept"].sum() > 0


def test_c4_default_mode(gpu, ora, c4_stream):
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384)
    sub = c4_stream.slice(0, 32 * 16384)
    ra = gpu.reorder_stream(ci, pl, sub, 32, inter=True)
    rb = ora.reorder_stream(co, pl, sub, 32, inter=True)
    _compare(ra, rb, "C4 default mode, 32 batches")


def test_c4_default_mode_dp_me_32(gpu, ora, c4_stream):
    """SURVEY §8(d) C4 second shape: DP_me = 32 (span 4 assembled sums)."""
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, 32, 1), (1, 128, 2), (1, 32, 1), 16384)
    sub = c4_stream.slice(0, 16 * 16384)
    ra = gpu.reorder_stream(ci, pl, sub, 16, inter=True)
    rb = ora.reorder_stream(co, pl, sub, 16, inter=True)
    _compare(ra, rb, "C4 default mode DP_me 32, 16 batches")


def test_c2_all_iterations(gpu, ora):
    model, cluster, book = H.llava_model(), H.a800_cluster(64), H.llava_book()
    ci, co = gpu.cost_model(model, cluster, book), ora.cost_model(model, cluster, book)
    pl = H.plan((1, 1, 1), (1, 1, 2), (1, 1, 1), 32)
    s = synth_stream(10000 * 32, seed=2024, family="skewed")
    ra = gpu.reorder_stream(ci, pl, s, 10000, inter=True)
    rb = ora.reorder_stream(co, pl, s, 10000, inter=True)
    _compare(ra, rb, "C2 10K iterations")


def test_c3_exact(gpu, ora):
    m, cl, bk = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
    st = stats_to_c(m.seq_len, 2048.0, 2048.0)
    ci, co = gpu.cost_model(m, cl, bk), ora.cost_model(m, cl, bk)
    g = gpu.model_orchestration(ci, st, 1920)
    r = ora.model_orchestration(co, st, 1920)
    assert g["best"] == r["best"] and g["times"] == r["times"], (g, r)
    assert g["candidates_evaluated"] == r["candidates_evaluated"] == 140370
    tuples = ora.enumerate_parallelism(cl, 1920)
    assert gpu.enumerate_parallelism(cl, 1920) == tuples
    rng = np.random.default_rng(3)
    sub = [tuples[i] for i in sorted(rng.choice(len(tuples), 2048, replace=False).tolist())]
    ca, cb = gpu.solve_subproblem(ci, st, sub, 1920), ora.solve_subproblem(co, st, sub, 1920)
    for x, y in zip(ca, cb):
        assert x == y, (x, y)


def test_c5_default_mode_chosen_plan(gpu, ora):
    """The search is compared live; the default-mode reorder of the batch
    (~2 min per reference call on one core) against the reference's recorded
    output (tests/golden/c5_default.npz, tests/golden/make_golden_c5.py)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    import make_golden_c5 as G5
    m, cl, bk, st, s = G5.c5_inputs()
    ci, co = gpu.cost_model(m, cl, bk), ora.cost_model(m, cl, bk)
    g, r = gpu.model_orchestration(ci, st, 16384), ora.model_orchestration(co, st, 16384)
    assert g["best"] == r["best"] and g["times"] == r["times"]
    want = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                "c5_default.npz"))
    best = g["best"]
    assert [best.encoder.pp, best.backbone.pp, best.generator.pp] == want["pp"].tolist()
    assert [best.encoder.dp, best.backbone.dp, best.generator.dp] == want["dp"].tolist()
    ra = gpu.reorder_stream(ci, best, s, 1, inter=True)
    _compare(ra, {k: want[k] for k in KEYS}, "C5 default mode, chosen plan")


def test_stats_full_stream(gpu, ora, c4_stream):
    """cost_size of every sample and compute_stats of a whole 1M-sample
    slice (integer-valued sums: exact in any order)."""
    sub = c4_stream.slice(0, 1 << 20)
    assert_same(gpu.cost_sizes(sub), ora.cost_sizes(sub), "cost_sizes")
    a, b = gpu.compute_stats(sub, 8192), ora.compute_stats(sub, 8192)
    assert (a.seq_len, a.mean_encoder_tokens, a.mean_generator_tokens) == \
        (b.seq_len, b.mean_encoder_tokens, b.mean_generator_tokens)


@pytest.mark.parametrize("bs,dp,inter,fam", [(32768, 128, False, "mixed"), (32768, 128, True, "dense"),
                                             (32768, 1024, False, "dense"), (20000, 100, False, "mixed")])
def test_beyond_fused_limits(gpu, ora, bs, dp, inter, fam):
    """Global batches beyond the fused kernels' 16,384 samples / 512 groups
    (the reference accepts any batch, src/reorder.cpp:319-396): the generic
    route (device radix sort + one-CTA greedy per batch)."""
    ci, co = _desk(gpu, ora)
    pl = H.plan((1, dp, 1), (1, dp, 2), (1, dp, 1), bs)
    s = synth_stream(2 * bs, seed=31, family=fam)
    ra = gpu.reorder_stream(ci, pl, s, 2, inter=inter)
    rb = ora.reorder_stream(co, pl, s, 2, inter=inter)
    _compare(ra, rb, f"BS {bs} DP {dp} inter {inter}")
