"""Parity cases shared by the oracle pinning tests (port vs compiled
reference, CPU) and the GPU parity tests (CUDA path vs oracle).

Every `check_*(impl, oracle, ...)` feeds identical inputs to both planners
and asserts BIT-EXACT equality: orders, assignments and plans are integers,
and every floating value is produced by the same IEEE operation sequence
(the north_star's 1e-6 relative slack is not needed and not used)."""
from __future__ import annotations

import numpy as np

from paper_2408_04275_b200.api import ASCENDING, DESCENDING, SampleBatch, stats_to_c
from paper_2408_04275_b200.workload import synth_stream

import helpers as H


def assert_same(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    if a.dtype.kind == "f":
        same = (a == b) | (np.isnan(a) & np.isnan(b))
        if not same.all():
            i = np.flatnonzero(~same.ravel())[0]
            raise AssertionError(f"{what}: first mismatch at {i}: {a.ravel()[i]!r} vs {b.ravel()[i]!r}"
                                 f" ({(~same).sum()} of {same.size})")
    else:
        if not np.array_equal(a, b):
            i = np.flatnonzero((a != b).ravel())[0]
            raise AssertionError(f"{what}: first mismatch at {i}: {a.ravel()[i]} vs {b.ravel()[i]}"
                                 f" ({(a != b).sum()} of {a.size})")


# ------------------------------------------------------------------ intra
def intra_size_sets(rng):
    yield np.array([1, 3, 2, 4.0]), 2
    yield np.array([2, 3, 4, 5.0]), 2
    yield np.full(12, 3.0), 4
    yield np.zeros(10), 3
    yield np.array([0.0, -0.0, 0.0, 5.0, -0.0]), 2
    for _ in range(20):
        n = int(rng.integers(1, 300))
        m = int(rng.integers(1, 20))
        kind = rng.integers(0, 4)
        if kind == 0:
            s = rng.lognormal(4.0, 0.8, n)
        elif kind == 1:
            s = 2.0 * rng.integers(0, 50, n)
        elif kind == 2:
            s = np.where(rng.random(n) < 0.35, 0.0, 2.0 * rng.integers(1, 4000, n))
        else:
            s = rng.integers(0, 3, n).astype(float)
        yield s.astype(float), m
    for n, m in ((512, 8), (2048, 64), (4096, 128)):
        yield 2.0 * synth_stream(n, int(rng.integers(1, 1 << 30)), "skewed").modality(), m


def check_intra(impl, oracle, rng):
    for sizes, m in intra_size_sets(rng):
        for order in (ASCENDING, DESCENDING):
            for eq in (False, True):
                a = impl.intra_partition(sizes, m, order, eq)
                b = oracle.intra_partition(sizes, m, order, eq)
                assert a.groups == b.groups, (len(sizes), m, order, eq)
        flat = oracle.intra_partition(sizes, m, ASCENDING, True).flat()
        if len(sizes) >= m:
            assert_same(impl.block_group_loads(sizes, flat, m),
                        oracle.block_group_loads(sizes, flat, m), "block loads")


def check_select(impl, oracle, rng):
    for _ in range(50):
        n = int(rng.integers(1, 40))
        keys = np.round(rng.lognormal(0, 0.7, n), int(rng.integers(0, 3)))
        pending = np.sort(rng.choice(n, int(rng.integers(1, n + 1)), replace=False))
        k = int(rng.integers(0, len(pending) + 1))
        assert impl.select_min(keys, pending, k) == oracle.select_min(keys, pending, k)
        target = float(rng.uniform(0, keys.sum()))
        assert (impl.select_closest(keys, pending, k, target)
                == oracle.select_closest(keys, pending, k, target))


# ---------------------------------------------------------------- schedule
def schedule_cases(rng):
    for p in range(1, 7):
        for l in range(1, 7):
            yield np.full((l, p), 0.7), np.full((l, p), 1.3), 1
    for _ in range(40):
        l = int(rng.integers(1, 40))
        p = int(rng.integers(1, 9))
        f, b = H.random_times(rng, l, p)
        yield f, b, 1
    for _ in range(20):
        vpp = int(rng.integers(2, 4))
        d = int(rng.integers(1, 4))
        p = d * vpp
        l = d * int(rng.integers(1, 6))
        f, b = H.random_times(rng, l, p)
        yield f, b, vpp


def check_schedule(impl, oracle, rng):
    for f, b, vpp in schedule_cases(rng):
        ta = impl.schedule(f, b, vpp)
        tb = oracle.schedule(f, b, vpp)
        assert ta.iteration_time == tb.iteration_time
        for fld in ("device", "microbatch", "stage", "phase", "start", "end", "device_busy"):
            assert_same(getattr(ta, fld), getattr(tb, fld), fld)
        ia, ib = impl.get_intervals(ta), oracle.get_intervals(tb)
        assert [(i.start, i.end, i.filled_by) for i in ia] == [(i.start, i.end, i.filled_by) for i in ib]
        if vpp == 1:
            assert_same(impl.interval_windows(f, b), oracle.interval_windows(f, b), "windows")
    # batched makespans
    for vpp, (l, p) in ((1, (32, 4)), (1, (7, 3)), (2, (8, 4))):
        f = rng.uniform(0.1, 2.0, (17, l, p))
        b = rng.uniform(0.1, 2.0, (17, l, p))
        ia, ba = impl.schedule_batch(f, b, vpp, with_busy=True)
        ib, bb = oracle.schedule_batch(f, b, vpp, with_busy=True)
        assert_same(ia, ib, "batch makespan")
        assert_same(ba, bb, "batch busy")


def check_exhaustive(impl, oracle, rng):
    """Every ordering's makespan (the reference's small-instance optimality
    oracle, tests/test_reorder.cpp:215-239), vpp 1 and 2, ties included."""
    cases = [(H.skewed_times(rng.lognormal(0, 0.5, 6), 3, 0.4), 1),
             (H.random_times(rng, 5, 4), 1),
             ((np.full((4, 2), 0.5), np.full((4, 2), 1.0)), 1),   # all orders tie
             (H.random_times(rng, 4, 4), 2),
             (H.random_times(rng, 1, 3), 1)]
    for (f, b), vpp in cases:
        ta, oa, aa = impl.exhaustive_order(f, b, vpp, with_all=True)
        tb, ob, ab = oracle.exhaustive_order(f, b, vpp, with_all=True)
        assert ta == tb and oa == ob, (f.shape, vpp, ta, tb, oa, ob)
        assert_same(aa, ab, "all orderings")
    f, b = H.skewed_times(rng.lognormal(0, 0.5, 8), 3, 0.4)   # 40,320 orderings
    ta, oa, _ = impl.exhaustive_order(f, b, 1)
    tb, ob, _ = oracle.exhaustive_order(f, b, 1)
    assert ta == tb and oa == ob


# ------------------------------------------------------------------- inter
def inter_cases(rng):
    for _ in range(30):
        l = int(rng.integers(1, 14))
        p = int(rng.integers(1, 6))
        enc = rng.lognormal(0, 0.6, l)
        f, b = H.skewed_times(enc, p, 0.3)
        yield f, b, f[:, 0].copy(), 1
    for _ in range(20):
        l = int(rng.integers(2, 40))
        p = int(rng.integers(2, 7))
        f, b = H.random_times(rng, l, p)
        yield f, b, rng.lognormal(0, 0.5, l), 1
    for _ in range(4):  # tie-heavy keys
        l, p = 24, 4
        f, b = H.random_times(rng, l, p)
        yield f, b, np.round(rng.uniform(0, 3, l)), 1
    for _ in range(12):
        vpp = int(rng.integers(2, 4))
        d = int(rng.integers(2, 4))
        l = d * int(rng.integers(1, 5))
        f, b = H.skewed_times(rng.lognormal(0, 0.5, l), d * vpp, 0.4)
        yield f, b, f[:, 0].copy(), vpp
    f, b = H.skewed_times(np.full(8, 0.7), 4, 0.4)
    yield f, b, np.full(8, 0.7), 2


def check_inter(impl, oracle, rng):
    for f, b, keys, vpp in inter_cases(rng):
        assert (impl.inter_reorder(f, b, keys, vpp)
                == oracle.inter_reorder(f, b, keys, vpp)), (f.shape, vpp)
    f = rng.uniform(0.1, 2.0, (9, 32, 4))
    b = 2.0 * f
    keys = f[:, :, 0].copy()
    assert_same(impl.inter_reorder_batch(f, b, keys, 1),
                oracle.inter_reorder_batch(f, b, keys, 1), "inter batch")


# -------------------------------------------------------------- cost model
def cost_models(impl, oracle):
    """(name, impl handle, oracle handle, plans) over several books."""
    cases = [
        ("desk", H.desk_model(), H.desk_cluster(64), H.desk_book()),
        ("toy-flat", H.toy_model(), H.toy_cluster(16), H.flat_book(0.4, 1.0, 0.4)),
        ("analytic", H.toy_model(), H.toy_cluster(16), H.Book(analytic_efficiency=0.5)),
        ("llava", H.llava_model(), H.a800_cluster(64), H.llava_book()),
    ]
    for name, model, cluster, book in cases:
        yield name, impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)


PLANS = [
    H.plan((1, 2, 1), (1, 2, 2), (1, 2, 1), 8),
    H.plan((1, 8, 1), (1, 8, 2), (1, 8, 1), 512),
    H.plan((2, 4, 1), (2, 8, 2), (1, 8, 1), 64),
    H.plan((1, 2, 1), (1, 4, 2), (1, 4, 1), 48, vpp=2),
    H.plan((1, 1, 1), (1, 2, 1), (1, 1, 1), 8),
]


def check_cost(impl, oracle, rng):
    for name, ci, co in cost_models(impl, oracle):
        for mod in range(3):
            for tp in (1, 2, 4, 8):
                loads = np.concatenate([[0.0, 8192.0, 9000.0, 1.5], rng.uniform(0, 10000, 20)])
                fa, ba = impl.unit_times(ci, mod, tp, loads)
                fb, bb = oracle.unit_times(co, mod, tp, loads)
                assert_same(fa, fb, f"{name} fwd")
                assert_same(ba, bb, f"{name} bwd")
        for pl in PLANS:
            l = 12
            enc = rng.integers(0, 20000, l)
            cnt = np.full(l, max(1, pl.samples_per_microbatch()))
            fa, ba = impl.build_stage_times(ci, pl, enc, enc, cnt)
            fb, bb = oracle.build_stage_times(co, pl, enc, enc, cnt)
            assert_same(fa, fb, f"{name} stage fwd")
            assert_same(ba, bb, f"{name} stage bwd")
            assert_same(impl.microbatch_fwd_keys(ci, pl, enc, enc, cnt),
                        oracle.microbatch_fwd_keys(co, pl, enc, enc, cnt), f"{name} keys")
            ma, mb = impl.memory_check(ci, pl), oracle.memory_check(co, pl)
            assert list(ma.bytes_per_gpu) == list(mb.bytes_per_gpu) and ma.pass_ == mb.pass_


# ------------------------------------------------------- disaggregated path
def disagg_cases(rng):
    yield H.plan((1, 8, 1), (1, 8, 2), (1, 8, 1), 512), "skewed"
    yield H.plan((1, 2, 1), (1, 8, 2), (1, 4, 1), 256), "mixed"
    yield H.plan((1, 2, 1), (1, 2, 2), (1, 2, 1), 8), "skewed"
    yield H.plan((1, 1, 1), (1, 2, 1), (1, 1, 1), 8), "skewed"
    yield H.plan((1, 2, 1), (1, 4, 2), (1, 4, 1), 64, vpp=2), "mixed"
    yield H.plan((1, 4, 1), (1, 4, 2), (1, 4, 1), 90), "mixed"  # n % m != 0 blocks
    # stage layouts of the compile-time tiled simulations and the generic one
    yield H.plan((1, 4, 2), (1, 4, 1), (1, 4, 1), 64), "mixed"
    yield H.plan((1, 4, 1), (1, 4, 1), (1, 4, 2), 64), "skewed"
    yield H.plan((1, 4, 1), (1, 4, 3), (1, 4, 2), 64), "mixed"
    yield H.plan((1, 8, 1), (1, 8, 6), (1, 8, 1), 1024), "mixed"  # l = 128, 4 chunks


def check_disaggregated(impl, oracle, rng, modes=None):
    modes = modes or [dict(intra=True, inter=True), dict(intra=True, inter=False),
                      dict(intra=True, inter=True, sort_order=DESCENDING),
                      dict(intra=False, inter=True)]
    model, cluster, book = H.desk_model(), H.desk_cluster(64), H.desk_book()
    ci, co = impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)
    cases = list(disagg_cases(rng))
    # a batch with oversized samples (> 32767 tokens: the kernel's 32-bit path)
    big = H.plan((1, 8, 1), (1, 8, 2), (1, 8, 1), 512)
    cases.append((big, "big"))
    for pl, fam in cases:
        if fam == "big":
            batch = synth_stream(pl.global_batch, 77, "skewed")
            batch.image_tokens[:5] = np.array([40000, 70000, 1, 33000, 123456], dtype=np.int32)
        else:
            batch = synth_stream(pl.global_batch, int(rng.integers(1, 1 << 30)), fam)
        for md in modes:
            ra = impl.disaggregated_reorder(ci, pl, batch, **md)
            rb = oracle.disaggregated_reorder(co, pl, batch, **md)
            tag = f"{pl} {md}"
            assert_same(ra.output_order, rb.output_order, tag + " order")
            assert_same(ra.group_load_before, rb.group_load_before, tag + " lb")
            assert_same(ra.group_load_after, rb.group_load_after, tag + " la")
            assert ra.t_iter_before == rb.t_iter_before, tag
            assert ra.t_iter_after == rb.t_iter_after, tag


STREAM_CASES = [  # (n_batches, bs, dp_lm, dp_me, pp triple, inter)
    (3, 512, 8, 8, (1, 2, 1), True),
    (37, 256, 8, 8, (1, 2, 1), False),     # CTAs of the simulations span batches
    (5, 4096, 8, 8, (1, 2, 1), False),     # l = 512: many staged chunks
    (4, 2048, 16, 4, (1, 2, 1), True),     # span 4: assembled microbatch sums
    (3, 1024, 8, 8, (2, 1, 1), True),
    (2, 16384, 128, 128, (1, 2, 1), False),  # BASELINE config 4 batch shape
    (40, 32, 1, 1, (1, 2, 1), True),      # BASELINE config 2 shape: one group of 32 per batch
    (6, 4096, 32, 32, (1, 2, 1), False, "dense"),   # greedy kept: counting scatter
    (4, 1000, 8, 8, (1, 2, 1), False, "dense"),     # n % 8 != 0: 32-bit path
    (5, 2048, 16, 16, (1, 2, 1), True, "dense"),
    (2, 4096, 8, 8, (1, 2, 1), True),      # l = 512 > 255: warp-per-problem inter
    (2, 1024, 4, 4, (2, 9, 3), True),      # p = 14 > 8: warp-per-problem inter
]


def check_stream(impl, oracle, rng, cases=None):
    model, cluster, book = H.desk_model(), H.desk_cluster(64), H.desk_book()
    ci, co = impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)
    for n_batches, bs, dp, dp_me, pp, inter, *fam in cases or STREAM_CASES:
        pl = H.plan((1, dp_me, pp[0]), (1, dp, pp[1]), (1, dp_me, pp[2]), bs)
        s = synth_stream(n_batches * bs, int(rng.integers(1, 1 << 30)), fam[0] if fam else "mixed")
        ra = impl.reorder_stream(ci, pl, s, n_batches, inter=inter)
        rb = oracle.reorder_stream(co, pl, s, n_batches, inter=inter)
        for k in ("output_order", "load_before", "load_after", "t_iter_before", "t_iter_after"):
            assert_same(ra[k], rb[k], f"{k} {n_batches}x{bs} dp {dp}/{dp_me} pp {pp}")


# vpp-1 plans beyond 8 stages: the warp-per-group simulations (register
# form for p <= 128, shared-memory form above), with ragged l < p and group
# counts that leave the last warps of a CTA idle
MANY_STAGE_PLANS = [
    H.plan((1, 2, 1), (1, 2, 11), (1, 2, 3), 8),     # p = 15
    H.plan((1, 2, 1), (1, 4, 71), (1, 2, 7), 16),    # p = 79 (BASELINE config 5 shape)
    H.plan((1, 2, 1), (1, 2, 100), (1, 2, 9), 8),    # p = 110 (4 stages per lane)
    H.plan((1, 2, 1), (1, 2, 140), (1, 2, 3), 8),    # p = 144 (shared-memory form)
]


def check_simulate(impl, oracle, rng):
    model, cluster, book = H.desk_model(), H.desk_cluster(1172), H.desk_book()
    ci, co = impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)
    for pl in PLANS + MANY_STAGE_PLANS:
        groups = []
        for g in range(int(rng.integers(1, 12 if pl in MANY_STAGE_PLANS else 5))):
            l = pl.microbatch_count() if pl.vpp > 1 else int(rng.integers(1, 20))
            enc = rng.integers(0, 9000, l)
            groups.append((enc, enc, np.full(l, max(1, pl.samples_per_microbatch()))))
        a = impl.simulate_iteration(ci, pl, groups)
        b = oracle.simulate_iteration(co, pl, groups)
        for k in a:
            assert_same(a[k], b[k], k)


# ------------------------------------------------ cost_size / compute_stats
def stats_batches(rng):
    """Sample batches for Sample::cost_size (core.hpp:160-167) and
    compute_stats (src/workload.cpp:206-220): both families, samples without
    any modality subsequence, image-only / audio-only samples, one sample,
    and large token counts (the 32-bit path's sums)."""
    yield synth_stream(4096, int(rng.integers(1, 1 << 30)), "mixed")
    yield synth_stream(777, int(rng.integers(1, 1 << 30)), "skewed")
    yield SampleBatch.from_lists([(5, [], [])])
    yield SampleBatch.from_lists([(1, [3, 4], [7]), (2, [], [9]), (0, [11], []), (3, [], [])])
    yield SampleBatch.from_lists([(10, [int(t)], [int(u)]) for t, u in
                                  zip(rng.integers(1, 1 << 20, 300), rng.integers(0, 1 << 20, 300))])


def check_stats(impl, oracle, rng):
    for batch in stats_batches(rng):
        assert_same(impl.cost_sizes(batch), oracle.cost_sizes(batch), f"cost_sizes n={batch.n}")
        for seq_len in (8192, 1):
            a, b = impl.compute_stats(batch, seq_len), oracle.compute_stats(batch, seq_len)
            assert (a.seq_len, a.mean_encoder_tokens, a.mean_generator_tokens) == \
                (b.seq_len, b.mean_encoder_tokens, b.mean_generator_tokens), (batch.n, seq_len)


# ------------------------------------------------------------ orchestration
def orch_cases():
    yield H.toy_model(), H.quiet_cluster(12), H.flat_book(1.0, 1.0, 1.0), 8, 1
    yield H.toy_model(), H.quiet_cluster(16), H.tp_scaled_book(0.3, 1.7, 0.9), 4, 1
    yield H.toy_model(), H.quiet_cluster(24), H.tp_scaled_book(0.4, 2.0, 0.6), 8, 2
    yield H.desk_model(), H.desk_cluster(64), H.desk_book(), 64, 1
    yield H.mllm72b_model(), H.a800_cluster(112), H.mllm72b_book(), 240, 1


def outcome(fn, *args):
    """Result, or (error class, message) — both sides must agree on either."""
    try:
        return fn(*args)
    except Exception as e:  # noqa: BLE001 — the error itself is the outcome
        return (type(e).__name__, str(e))


def check_brute(impl, oracle, rng):
    """brute_force_oracle and rigid_baseline (src/orchestrator.cpp:407-491):
    plan, times and the evaluated count; the cap and infeasible errors."""
    from paper_2408_04275_b200.api import CapExceededError
    cases = [(H.toy_model(), H.quiet_cluster(12), H.flat_book(1.0, 1.0, 1.0), 8, 1),
             (H.toy_model(), H.quiet_cluster(16), H.tp_scaled_book(0.3, 1.7, 0.9), 4, 1),
             (H.toy_model(), H.quiet_cluster(24), H.tp_scaled_book(0.4, 2.0, 0.6), 8, 2),
             (H.desk_model(), H.desk_cluster(32), H.desk_book(), 64, 1)]
    for model, cluster, book, bs, vpp in cases:
        ci, co = impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)
        stats = stats_to_c(model.seq_len, 1000.0, 1000.0)
        a = outcome(impl.brute_force_oracle, ci, stats, bs, vpp)
        b = outcome(oracle.brute_force_oracle, co, stats, bs, vpp)
        assert a == b, (a, b)
        a = outcome(impl.rigid_baseline, ci, stats, bs, vpp)
        b = outcome(oracle.rigid_baseline, co, stats, bs, vpp)
        assert a == b, (a, b)
    # the cap: same error class and text
    model, cluster, book = H.desk_model(), H.desk_cluster(64), H.desk_book()
    ci, co = impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)
    stats = stats_to_c(model.seq_len, 1000.0, 1000.0)
    msgs = []
    for pl, c in ((impl, ci), (oracle, co)):
        try:
            pl.brute_force_oracle(c, stats, 64)
            raise AssertionError("cap not enforced")
        except CapExceededError as e:
            msgs.append(str(e))
    assert msgs[0] == msgs[1], msgs


def check_orchestration(impl, oracle, rng):
    for model, cluster, book, bs, vpp in orch_cases():
        ci, co = impl.cost_model(model, cluster, book), oracle.cost_model(model, cluster, book)
        stats = stats_to_c(model.seq_len, 1000.0, 1000.0)
        ta = impl.enumerate_parallelism(cluster, bs)
        tb = oracle.enumerate_parallelism(cluster, bs)
        assert ta == tb
        sub = [tb[i] for i in sorted(set(rng.integers(0, len(tb), 200).tolist()))]
        ca = impl.solve_subproblem(ci, stats, sub, bs, vpp)
        cb = oracle.solve_subproblem(co, stats, sub, bs, vpp)
        for x, y in zip(ca, cb):
            assert x == y, (x, y)
        ra = impl.model_orchestration(ci, stats, bs, vpp)
        rb = oracle.model_orchestration(co, stats, bs, vpp)
        assert ra["best"] == rb["best"] and ra["times"] == rb["times"]
        assert ra["candidates_evaluated"] == rb["candidates_evaluated"]
        plans = [c.plan for c in cb if c.feasible][:50]
        if plans:
            assert impl.predict_times(ci, stats, plans) == oracle.predict_times(co, stats, plans)
