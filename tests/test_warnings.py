"""Warning log: the strings the reference's CostModel appends to its warning
sink (CostModel::set_warning_sink, include/cost_model.hpp:147; texts of
src/cost_model.cpp:84-95 and :248-251), in the reference's query order
(SURVEY.md §8(b) "Warnings").

CPU: the compiled reference's C shim (oracle/_ref) against the reference's
own known answers (tests/test_cost_model.cpp:26-36, :259-273).
GPU: the product's log against the compiled reference, string for string,
for every covered call — including whole disaggregated_reorder / stream
calls, where the queries come from microbatch token sums on the device.
"""
import numpy as np
import pytest

import helpers as H
from paper_2408_04275_b200.api import (ALLOWED_TP, BACKBONE, DESCENDING, ENCODER, GENERATOR,
                                       Book)
from paper_2408_04275_b200.workload import synth_stream


def narrow_book(lo=600.0, hi=2500.0, generator_rows=False) -> Book:
    """Profile rows only inside [lo, hi] token loads (so microbatch means
    clamp on both sides); the generator has no rows unless asked (analytic
    fallback warnings)."""
    b = Book()
    b.analytic_efficiency = 0.5
    units = [ENCODER, BACKBONE] + ([GENERATOR] if generator_rows else [])
    for u in units:
        for tp in ALLOWED_TP:
            b.add_row(u, tp, lo, 0.01 * tp, 0.02 * tp)
            b.add_row(u, tp, hi, 0.05 * tp, 0.10 * tp)
    return b


def _model(seq_len=4096):
    m = H.desk_model()
    m.seq_len = seq_len
    return m


def _fresh(pl, on=True):
    pl.warnings_enable(on)


def _ref(ref):
    if not ref.lib.has("warnings_enable"):
        pytest.skip("compiled reference shim without the warning log")
    return ref


# ------------------------------------------------------------------ CPU
def test_ref_known_answers(ref):
    """tests/test_cost_model.cpp:26-36 (clamp with warning, exact key and
    midpoint without) and :259-273 (analytic fallback, one warning)."""
    r = _ref(ref)
    b = Book()
    b.add_row(ENCODER, 8, 2048.0, 0.5)
    b.add_row(ENCODER, 8, 8192.0, 2.0)
    b.analytic_efficiency = 0.5
    cm = r.cost_model(_model(), H.desk_cluster(64), b)
    _fresh(r)
    f, _ = r.unit_times(cm, ENCODER, 8, [4096.0, 6144.0])
    assert r.warnings() == []
    r.unit_times(cm, ENCODER, 8, [10000.0])
    assert r.warnings()[0] == "token load 10000.000000 above profile range; clamped"
    _fresh(r)
    r.unit_times(cm, GENERATOR, 1, [1000.0])
    w = r.warnings()
    assert w and w[0] == "module 'generator' has no profile; using analytic estimate"
    _fresh(r, False)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_unit_times_and_stage_queries(gpu, ref):
    r = _ref(ref)
    model, cluster, book = _model(), H.desk_cluster(64), narrow_book()
    cg, cr = gpu.cost_model(model, cluster, book), r.cost_model(model, cluster, book)
    rng = np.random.default_rng(5)
    loads = np.concatenate([[0.0, 600.0, 2500.0, 599.999, 2500.5], rng.uniform(0, 4000, 60)])
    for u in (ENCODER, BACKBONE, GENERATOR):
        for pl in (gpu, r):
            _fresh(pl)
        a = gpu.unit_times(cg, u, 2, loads)
        bref = r.unit_times(cr, u, 2, loads)
        assert np.array_equal(a[0], bref[0]) and np.array_equal(a[1], bref[1])
        assert gpu.warnings() == r.warnings(), u
    plan = H.plan((1, 4, 1), (2, 8, 2), (1, 2, 1), 64)
    enc = rng.integers(0, 9000, 40)
    gen = rng.integers(0, 9000, 40)
    cnt = rng.integers(1, 6, 40)
    for pl in (gpu, r):
        _fresh(pl)
    gpu.build_stage_times(cg, plan, enc, gen, cnt)
    r.build_stage_times(cr, plan, enc, gen, cnt)
    gpu.microbatch_fwd_keys(cg, plan, enc, gen, cnt)
    r.microbatch_fwd_keys(cr, plan, enc, gen, cnt)
    groups = [(enc[i:i + 8], gen[i:i + 8], cnt[i:i + 8]) for i in range(0, 40, 8)]
    gpu.simulate_iteration(cg, plan, groups)
    r.simulate_iteration(cr, plan, groups)
    wg, wr = gpu.warnings(), r.warnings()
    assert len(wr) > 100 and wg == wr
    for pl in (gpu, r):
        _fresh(pl, False)


@pytest.mark.gpu
@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("dims", [((1, 8, 1), (1, 8, 2), (1, 8, 1)),    # span 1
                                  ((1, 2, 1), (1, 8, 2), (1, 4, 1))])   # span 4 (assembled)
def test_reorder_calls(gpu, ref, inter, dims):
    """Whole disaggregated_reorder and stream calls: before / intra / after
    microbatch phases, per batch, in the reference's order."""
    r = _ref(ref)
    bs, nb = 512, 4
    model, cluster = _model(), H.desk_cluster(64)
    book = narrow_book(generator_rows=dims[0][1] == 2)
    cg, cr = gpu.cost_model(model, cluster, book), r.cost_model(model, cluster, book)
    plan = H.plan(*dims, bs)
    s = synth_stream(nb * bs, seed=17, family="mixed")
    for pl in (gpu, r):
        _fresh(pl)
    one_g = gpu.disaggregated_reorder(cg, plan, s.slice(0, bs), inter=inter)
    one_r = r.disaggregated_reorder(cr, plan, s.slice(0, bs), inter=inter)
    assert np.array_equal(one_g.output_order, one_r.output_order)
    w1g, w1r = gpu.warnings(), r.warnings()
    assert len(w1r) > 0 and w1g == w1r
    for pl in (gpu, r):
        _fresh(pl)
    for order in (0, DESCENDING):
        gpu.reorder_stream(cg, plan, s, nb, inter=inter, sort_order=order)
        r.reorder_stream(cr, plan, s, nb, inter=inter, sort_order=order)
    wg, wr = gpu.warnings(), r.warnings()
    assert len(wr) > len(w1r) and wg == wr
    for pl in (gpu, r):
        _fresh(pl, False)
