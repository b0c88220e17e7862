"""Known-answer tests restated from the reference's own unit tests
(proj/tests/test_reorder.cpp, test_pipeline_sim.cpp, test_orchestrator.cpp,
test_cost_model.cpp).  Each `golden_*(planner)` runs against any backend:
the oracles on CPU (tests/test_oracle_golden.py) and the CUDA path on a B200
(tests/test_gpu_golden.py)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2408_04275_b200 import api as A

import helpers as H

approx = lambda v, rel=1e-12: pytest.approx(v, rel=rel, abs=1e-12)


def golden_intra(pl):
    # test_reorder.cpp:63-77
    sizes = [1, 3, 2, 4]
    order = pl.intra_reorder_order(sizes, 2)
    assert [sizes[i] for i in order] == [1, 3, 2, 4]
    lpt = pl.intra_partition(sizes, 2, A.DESCENDING)
    assert lpt.loads(sizes) == [5.0, 5.0]
    # test_reorder.cpp:79-84
    sizes = [2, 3, 4, 5]
    part = pl.intra_partition(sizes, 2)
    assert [sizes[i] for i in part.flat()] == [2, 4, 3, 5]
    assert part.max_load(sizes) == 8.0
    # test_reorder.cpp:86-94
    sizes = [3.0] * 12
    for m in (1, 2, 3, 4):
        for load in pl.intra_partition(sizes, m).loads(sizes):
            assert load == approx(3.0 * 12 / m)
    with pytest.raises(A.InternalError):
        pl.intra_partition([], 2)
    with pytest.raises(A.InternalError):
        pl.intra_partition([1.0], 0)


def golden_select(pl):
    # test_reorder.cpp:139-158
    assert pl.select_min([5, 1, 3], [0, 1, 2], 2) == [1, 2]
    with pytest.raises(A.KTooLargeError):
        pl.select_min([5, 1, 3], [0, 1, 2], 4)
    assert pl.select_closest([5, 1, 3], [0, 1, 2], 1, 2.9) == [2]
    assert pl.select_closest([5, 1, 3, 2], [0, 1, 2, 3], 2, 4.0) == [2, 1]
    with pytest.raises(A.KTooLargeError):
        pl.select_closest([5, 1, 3], [0, 1, 2], 5, 1.0)


def golden_schedule(pl):
    # test_pipeline_sim.cpp:42-49
    tl = pl.schedule_1f1b([[1.0]], [[2.0]])
    assert tl.iteration_time == approx(3.0) and len(tl.start) == 2
    # :51-61 closed form (l + p - 1)(tf + tb)
    for p in range(1, 7):
        for l in range(1, 7):
            tl = pl.schedule_1f1b(np.full((l, p), 0.7), np.full((l, p), 1.3))
            assert tl.iteration_time == approx((l + p - 1) * 2.0)
    # :147-167 hand-enumerated interleaved schedule, one device, two chunks
    tl = pl.schedule_interleaved(np.ones((2, 2)), np.ones((2, 2)), 2)
    assert len(tl.start) == 8
    expect = [(0, 0, 0), (0, 1, 0), (0, 1, 1), (1, 0, 0), (0, 0, 1), (1, 1, 0),
              (1, 1, 1), (1, 0, 1)]
    for i, (mb, st, ph) in enumerate(expect):
        assert tl.start[i] == approx(float(i))
        assert (tl.microbatch[i], tl.stage[i], tl.phase[i]) == (mb, st, ph)
    assert tl.iteration_time == approx(8.0)
    # :169-174 indivisible vpp
    with pytest.raises(A.IndivisibleVppError):
        pl.schedule_interleaved(np.ones((4, 3)), np.ones((4, 3)), 2)
    with pytest.raises(A.IndivisibleVppError):
        pl.schedule_interleaved(np.ones((3, 4)), np.ones((3, 4)), 2)
    # :176-195 homogeneous intervals
    p, l = 4, 6
    iv = pl.get_intervals(pl.schedule_1f1b(np.ones((l, p)), np.ones((l, p))))
    assert len(iv) == l
    assert len(iv[0].filled_by) == p - 1
    for i in range(1, l - p + 1):
        assert len(iv[i].filled_by) == 1
    for i in range(l - p + 1, l):
        assert iv[i].filled_by == []
    for i in range(2, l - p + 1):
        assert iv[i].volume() == approx(iv[1].volume())
    # :281-297 bubble fractions via busy time
    tl = pl.schedule_1f1b(np.ones((4, 4)), np.ones((4, 4)))
    bub = (tl.device_idle().sum()) / (tl.device_count * tl.iteration_time)
    assert bub == approx(3 / 7)
    # negative stage times are rejected (pipeline_sim.cpp:214-230)
    with pytest.raises(A.InternalError):
        pl.schedule_1f1b([[-1.0]], [[1.0]])


def golden_cost(pl):
    model, cluster = H.toy_model(), H.toy_cluster(8)
    # test_cost_model.cpp:26-43 interpolation (TP 8 rows 4096->1, 8192->2)
    book = A.Book().add_row(A.ENCODER, 8, 4096, 1.0).add_row(A.ENCODER, 8, 8192, 2.0)
    cm = pl.cost_model(model, cluster, book)
    f, _ = pl.unit_times(cm, A.ENCODER, 8, [4096, 6144, 10000, 0.0, 5000])
    assert list(f[:4]) == [1.0, 1.5, 2.0, 1.0]
    assert f[4] == approx(1.0 + (5000 - 4096) / 4096)
    # :59-66 missing TP rows
    with pytest.raises(A.EmptyProfileError):
        pl.unit_times(cm, A.ENCODER, 4, [4096])
    # :68-77 backward defaults to 2x forward, rowwise
    book = A.Book().add_row(A.ENCODER, 2, 1024, 0.3).add_row(A.ENCODER, 2, 2048, 0.5, 1.4)
    cm = pl.cost_model(model, cluster, book)
    _, b = pl.unit_times(cm, A.ENCODER, 2, [1024, 2048, 1536])
    assert b[0] == approx(0.6) and b[1] == approx(1.4) and b[2] == approx(1.0)
    # :107-138 stage time with DP coupling
    book = (A.Book().add_row(A.ENCODER, 1, 0, 0.4, 0.8).add_row(A.BACKBONE, 1, 0, 2.0, 4.0)
            .add_row(A.GENERATOR, 1, 0, 0.6, 1.2))
    cm = pl.cost_model(model, cluster, book)
    plan = H.plan((1, 2, 1), (1, 4, 1), (1, 4, 1), 8)
    f, _ = pl.build_stage_times(cm, plan, [50], [50], [1])
    assert f[0, 0] == approx(0.8 + 2.0 * 512 * 50 * 2 / 300e9)  # stage + comm
    # :200-224 memory accounting 21e9
    m2 = H.toy_model()
    m2.backbone.param_grad_bytes, m2.backbone.optimizer_bytes, m2.backbone.activation_bytes_per_mb = 80e9, 160e9, 2e9
    c2 = H.toy_cluster(32)
    c2.gpu_mem_bytes = 100e9
    cm = pl.cost_model(m2, c2, H.flat_book(1, 1, 1))
    rep = pl.memory_check(cm, H.plan((1, 1, 1), (2, 2, 4), (1, 1, 1), 4))
    assert rep.bytes_per_gpu[1] == approx(21e9) and rep.fits[1] == 1
    # :244-257 frozen modules
    m3 = H.toy_model()
    m3.generator.frozen = True
    cm = pl.cost_model(m3, cluster, A.Book().add_row(A.GENERATOR, 1, 0, 0.6, 1.2))
    f, b = pl.unit_times(cm, A.GENERATOR, 1, [0.0])
    assert b[0] == approx(1.2 / 3.0) and f[0] == approx(0.6)
    # :259-273 analytic fallback
    cm = pl.cost_model(model, cluster, A.Book(analytic_efficiency=0.5))
    f, _ = pl.unit_times(cm, A.ENCODER, 1, [1000.0])
    params = 8 * (512.0 * 512.0 * (2.0 + 2.0 * 8 / 8) + 3.0 * 512 * 2048)
    assert f[0] == approx(2.0 * params * 1000 / (312e12 * 0.5))
    # add_row validation (cost_model.cpp:39-48)
    with pytest.raises(A.ConfigError):
        pl.cost_model(model, cluster, A.Book().add_row(A.ENCODER, 3, 0, 1.0))
    with pytest.raises(A.ConfigError):
        pl.cost_model(model, cluster, A.Book().add_row(A.ENCODER, 1, 0, -1.0))


def _stats(model):
    return A.stats_to_c(model.seq_len, 1000.0, 1000.0)


def golden_orchestration(pl):
    model = H.toy_model()
    st = _stats(model)
    # test_orchestrator.cpp:47-60
    cm = pl.cost_model(model, H.quiet_cluster(8), H.flat_book(0.4, 2.0, 0.6))
    t = pl.predict_times(cm, st, [H.plan((1, 2, 1), (1, 2, 2), (1, 2, 1), 2)])[0]
    assert t[1] == approx(0.0) and t[2] == approx(t[0])
    # :62-76
    cm = pl.cost_model(model, H.quiet_cluster(3), H.flat_book(0.5, 0.5, 0.5))
    t = pl.predict_times(cm, st, [H.plan((1, 1, 1), (1, 1, 1), (1, 1, 1), 9)])[0]
    assert t[1] == approx(8.0 * 1.5) and t[0] == approx(3.0 * 1.5)
    # :119-145 enumeration vs an independent count
    cluster = H.quiet_cluster(16)
    expect = 0
    for tp_me in (1, 2, 4, 8):
        for tp_lm in (1, 2, 4, 8):
            for tp_mg in (1, 2, 4, 8):
                for dp_lm in range(1, 9):
                    if 8 % dp_lm or tp_lm * dp_lm > 16:
                        continue
                    for dp_me in range(1, dp_lm + 1):
                        if dp_lm % dp_me or tp_me * dp_me > 16:
                            continue
                        for dp_mg in range(1, dp_lm + 1):
                            if dp_lm % dp_mg or tp_mg * dp_mg > 16:
                                continue
                            if tp_me * dp_me + tp_lm * dp_lm + tp_mg * dp_mg > 16:
                                continue
                            expect += 1
    tuples = pl.enumerate_parallelism(cluster, 8)
    assert len(tuples) == expect == len(set(tuples)) and tuples == sorted(tuples)
    assert {t[3] for t in pl.enumerate_parallelism(H.quiet_cluster(64), 7)} == {1, 7}
    # :147-161 symmetric split
    cm = pl.cost_model(model, H.quiet_cluster(12), H.flat_book(1.0, 1.0, 1.0))
    r = pl.solve_subproblem(cm, st, [(1, 1, 1, 1, 1, 1)], 8)[0]
    assert r.feasible and r.cont == pytest.approx((4.0, 4.0, 4.0), rel=1e-6)
    assert (r.plan.encoder.gpus(), r.plan.backbone.gpus(), r.plan.generator.gpus()) == (4, 4, 4)
    # :163-180 waterfilling
    cm = pl.cost_model(model, H.quiet_cluster(12), H.flat_book(1.0, 3.0, 1e-7))
    r = pl.solve_subproblem(cm, st, [(1, 1, 1, 1, 1, 1)], 4)[0]
    assert r.cont == pytest.approx((2.75, 8.25, 1.0), rel=1e-3)
    # :207-216 three GPUs force the singleton plan
    cm = pl.cost_model(model, H.quiet_cluster(3), H.flat_book(0.4, 2.0, 0.6))
    res = pl.model_orchestration(cm, st, 1)
    assert res["best"].total_gpus() == 3
    # :349-356 infeasible memory floors
    m4 = H.toy_model()
    m4.backbone.param_grad_bytes = m4.backbone.optimizer_bytes = 1e15
    m4.backbone.activation_bytes_per_mb = 1e9
    cm = pl.cost_model(m4, H.quiet_cluster(8), H.flat_book(0.4, 2.0, 0.6))
    with pytest.raises(A.InfeasibleError):
        pl.model_orchestration(cm, st, 4)


def golden_disaggregated(pl):
    model = H.toy_model()
    cm = pl.cost_model(model, H.toy_cluster(8), H.flat_book(0.4, 1.0, 0.4))
    # test_reorder.cpp:285-307 single group: loads before == after
    batch = A.SampleBatch.from_lists([(100, [10 * (i + 1)]) for i in range(6)])
    r = pl.disaggregated_reorder(cm, H.plan((1, 1, 1), (1, 1, 2), (1, 1, 1), 6), batch,
                                 inter=False)
    assert len(r.group_load_before) == 1
    assert r.group_load_after[0] == approx(r.group_load_before[0])
    # :361-370 batch size mismatch
    with pytest.raises(A.BatchSizeMismatchError):
        pl.disaggregated_reorder(cm, H.plan((1, 1, 1), (1, 1, 1), (1, 1, 1), 4),
                                 A.SampleBatch.from_lists([(10, [])]))
    # :309-359 balance + permutation over random batches
    rng = np.random.default_rng(83)
    plan = H.plan((1, 2, 1), (1, 2, 2), (1, 2, 1), 8)
    for _ in range(20):
        batch = A.SampleBatch.from_lists([(50, [int(10 + rng.integers(0, 500))]) for _ in range(8)])
        r = pl.disaggregated_reorder(cm, plan, batch)
        assert max(r.group_load_after) <= max(r.group_load_before) + 1e-9
        assert sorted(r.output_order.tolist()) == list(range(8))


ALL = [golden_intra, golden_select, golden_schedule, golden_cost, golden_orchestration,
       golden_disaggregated]
