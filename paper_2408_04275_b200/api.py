"""Python mirror of the reference planner API (mmplan, /root/reference/proj/core)
over the C ABI of include/disttrain_b200.h.

`Planner(lib)` exposes the reference entry points with the same names,
argument meaning and error classes (include/errors.hpp:22-84), so tests read
like the reference's own (proj/tests/test_*.cpp).  The product planner binds
libdisttrain_b200.so (CUDA, sm_100a); the oracles under oracle/ bind the same
class to the reference/port libraries for parity checks.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _capi as A
from ._capi import ptr

ENCODER, BACKBONE, GENERATOR = 0, 1, 2
ASCENDING, DESCENDING = 0, 1
FORWARD, BACKWARD = 0, 1
ALLOWED_TP = (1, 2, 4, 8)


# --------------------------------------------------------------- errors
class MmplanError(Exception):
    pass


class ConfigError(MmplanError):
    pass


class EmptyProfileError(ConfigError):
    pass


class InfeasibleError(MmplanError):
    pass


class InternalError(MmplanError):
    pass


class KTooLargeError(MmplanError):
    pass


class CapExceededError(MmplanError):
    pass


class IndivisibleVppError(MmplanError):
    pass


class BatchSizeMismatchError(MmplanError):
    pass


class InvalidArgument(MmplanError):
    pass


class TraceError(ConfigError):
    """TraceError (errors.hpp:35-47): kind() "ParseError" or
    "InvariantViolation" and the 1-based line()."""

    def __init__(self, msg, kind="", line=0):
        super().__init__(msg)
        self._kind = kind
        self._line = line

    def kind(self):
        return self._kind

    def line(self):
        return self._line


class CudaError(MmplanError):
    pass


_ERRORS = {1: InternalError, 2: KTooLargeError, 3: IndivisibleVppError,
           4: BatchSizeMismatchError, 5: ConfigError, 6: EmptyProfileError,
           7: InfeasibleError, 8: CapExceededError, 9: TraceError, 100: InvalidArgument,
           101: CudaError}

REASON_TEXT = {
    0: "",
    1: "dp does not divide the global batch",
    2: "activation memory of encoder exceeds GPU capacity at any allocation",
    3: "activation memory of backbone exceeds GPU capacity at any allocation",
    4: "activation memory of generator exceeds GPU capacity at any allocation",
    5: "memory floor exceeds the cluster",
    6: "no integer stage split is feasible",
}


# ------------------------------------------------------------ domain types
@dataclass
class Module:
    layers: int = 0
    hidden: int = 0
    ffn_hidden: int = 0
    heads: int = 0
    groups: int = 0
    param_grad_bytes: float = 0.0
    optimizer_bytes: float = 0.0
    activation_bytes_per_mb: float = 0.0
    frozen: bool = False


@dataclass
class Model:
    encoder: Module = field(default_factory=Module)
    backbone: Module = field(default_factory=Module)
    generator: Module = field(default_factory=Module)
    seq_len: int = 8192
    frozen_backward_factor: float = 1.0 / 3.0
    dp_sync_seconds: float = 0.0

    def to_c(self) -> A.ModelSpec:
        m = A.ModelSpec()
        for u, mod in enumerate((self.encoder, self.backbone, self.generator)):
            s = m.unit[u]
            s.arch.layers, s.arch.hidden, s.arch.ffn_hidden = mod.layers, mod.hidden, mod.ffn_hidden
            s.arch.heads, s.arch.groups = mod.heads, mod.groups
            s.mem.param_grad_bytes = mod.param_grad_bytes
            s.mem.optimizer_bytes = mod.optimizer_bytes
            s.mem.activation_bytes_per_mb = mod.activation_bytes_per_mb
            s.frozen = int(mod.frozen)
        m.seq_len = self.seq_len
        m.frozen_backward_factor = self.frozen_backward_factor
        m.dp_sync_seconds = self.dp_sync_seconds
        return m


@dataclass
class Cluster:
    total_gpus: int = 0
    gpus_per_node: int = 8
    peak_flops: float = 0.0
    gpu_mem_bytes: float = 0.0
    intra_node_bw: float = 0.0
    inter_node_bw: float = 0.0

    def to_c(self) -> A.ClusterSpec:
        return A.ClusterSpec(self.total_gpus, self.gpus_per_node, self.peak_flops,
                             self.gpu_mem_bytes, self.intra_node_bw, self.inter_node_bw)


@dataclass
class Book:
    """CostBook as the ordered list of add_row calls (cost_model.hpp:44)."""
    rows: list = field(default_factory=list)  # (module, tp, load, fwd, bwd|None)
    analytic_efficiency: float = 0.45
    analytic_bwd_fwd_ratio: float = 2.0

    def add_row(self, module, tp, token_load, fwd_s, bwd_s=None):
        self.rows.append((module, tp, float(token_load), float(fwd_s),
                          None if bwd_s is None else float(bwd_s)))
        return self


@dataclass(frozen=True)
class Choice:
    tp: int = 1
    dp: int = 1
    pp: int = 1

    def gpus(self):
        return self.tp * self.dp * self.pp


@dataclass(frozen=True)
class PlanSpec:
    encoder: Choice = Choice()
    backbone: Choice = Choice()
    generator: Choice = Choice()
    global_batch: int = 1
    vpp: int = 1

    def to_c(self) -> A.Plan:
        p = A.Plan()
        for u, c in enumerate((self.encoder, self.backbone, self.generator)):
            p.unit[u].tp, p.unit[u].dp, p.unit[u].pp = c.tp, c.dp, c.pp
        p.vpp = self.vpp
        p.global_batch = self.global_batch
        return p

    @staticmethod
    def from_c(p: A.Plan) -> "PlanSpec":
        ch = [Choice(p.unit[u].tp, p.unit[u].dp, p.unit[u].pp) for u in range(3)]
        return PlanSpec(ch[0], ch[1], ch[2], int(p.global_batch), int(p.vpp))

    def total_gpus(self):
        return self.encoder.gpus() + self.backbone.gpus() + self.generator.gpus()

    def microbatch_count(self):
        return self.global_batch // self.backbone.dp

    def samples_per_microbatch(self):
        return self.backbone.dp // self.encoder.dp

    def pipeline_devices(self):
        return self.encoder.pp + self.backbone.pp + self.generator.pp

    def virtual_stages(self):
        return self.pipeline_devices() * self.vpp


@dataclass
class SampleBatch:
    """CSR span of Samples (core.hpp:155): int32 tokens, absolute offsets."""
    text: np.ndarray
    image_offsets: np.ndarray
    image_tokens: np.ndarray
    audio_offsets: np.ndarray
    audio_tokens: np.ndarray

    @property
    def n(self):
        return len(self.image_offsets) - 1

    @staticmethod
    def from_lists(samples: Sequence) -> "SampleBatch":
        """samples: iterable of (text, [image tokens], [audio tokens])."""
        text, io, it, ao, at = [], [0], [], [0], []
        for s in samples:
            t, imgs = s[0], s[1]
            auds = s[2] if len(s) > 2 else []
            text.append(t)
            it.extend(imgs)
            io.append(len(it))
            at.extend(auds)
            ao.append(len(at))
        i32 = lambda v: np.ascontiguousarray(np.asarray(v, dtype=np.int32))
        return SampleBatch(i32(text), i32(io), i32(it), i32(ao), i32(at))

    def to_c(self) -> A.Samples:
        keep = [self.text, self.image_offsets, self.image_tokens,
                self.audio_offsets, self.audio_tokens]
        s = A.Samples(self.n, ptr(self.text, C.c_int32),
                      ptr(self.image_offsets, C.c_int32),
                      ptr(_nonempty(self.image_tokens), C.c_int32),
                      ptr(self.audio_offsets, C.c_int32),
                      ptr(_nonempty(self.audio_tokens), C.c_int32))
        s._keep = keep
        return s

    def slice(self, begin: int, end: int) -> "SampleBatch":
        io = self.image_offsets[begin:end + 1]
        ao = self.audio_offsets[begin:end + 1]
        return SampleBatch(
            np.ascontiguousarray(self.text[begin:end]),
            np.ascontiguousarray(io - io[0]),
            np.ascontiguousarray(self.image_tokens[io[0]:io[-1]]),
            np.ascontiguousarray(ao - ao[0]),
            np.ascontiguousarray(self.audio_tokens[ao[0]:ao[-1]]))

    def modality(self) -> np.ndarray:
        """Per-sample modality tokens (numpy, host-side helper for tests)."""
        ci = np.concatenate([[0], np.cumsum(self.image_tokens, dtype=np.int64)])
        ca = np.concatenate([[0], np.cumsum(self.audio_tokens, dtype=np.int64)])
        return (ci[self.image_offsets[1:]] - ci[self.image_offsets[:-1]]
                + ca[self.audio_offsets[1:]] - ca[self.audio_offsets[:-1]])


def _nonempty(a):
    return a if a.size else np.zeros(1, dtype=a.dtype)


@dataclass
class IntraPartition:
    groups: list

    def flat(self):
        return [i for g in self.groups for i in g]

    def loads(self, sizes):
        out = []
        for g in self.groups:
            acc = 0.0
            for i in g:
                acc += float(sizes[i])
            out.append(acc)
        return out

    def max_load(self, sizes):
        return max(self.loads(sizes))


@dataclass
class Timeline:
    device: np.ndarray
    microbatch: np.ndarray
    stage: np.ndarray
    phase: np.ndarray
    start: np.ndarray
    end: np.ndarray
    iteration_time: float
    device_busy: np.ndarray
    device_count: int
    microbatch_count: int
    stage_count: int

    def device_idle(self):
        return self.iteration_time - self.device_busy


@dataclass
class Interval:
    start: float
    end: float
    filled_by: list

    def volume(self):
        return self.end - self.start


@dataclass
class ReorderReport:
    output_order: np.ndarray
    group_load_before: np.ndarray
    group_load_after: np.ndarray
    t_iter_before: float
    t_iter_after: float


@dataclass
class Candidate:
    tuple: tuple
    feasible: bool
    infeasible_reason: str
    plan: PlanSpec
    times: tuple
    cont: tuple
    cont_t_iter: float

    @staticmethod
    def from_c(c: A.Candidate) -> "Candidate":
        t = c.tuple
        return Candidate((t.tp_me, t.dp_me, t.tp_lm, t.dp_lm, t.tp_mg, t.dp_mg),
                         bool(c.feasible), REASON_TEXT.get(c.reason, "?"),
                         PlanSpec.from_c(c.plan),
                         (c.times.t_warm, c.times.t_steady, c.times.t_iter),
                         (c.cont_x, c.cont_y, c.cont_z), c.cont_t_iter)


def tuple_to_c(t) -> A.Tuple:
    return A.Tuple(*[int(v) for v in t])


def stats_to_c(seq_len, mean_enc, mean_gen) -> A.WorkloadStats:
    return A.WorkloadStats(int(seq_len), float(mean_enc), float(mean_gen))


def microbatches_to_c(enc, gen, count):
    enc = np.ascontiguousarray(enc, dtype=np.int64)
    gen = np.ascontiguousarray(gen, dtype=np.int64)
    count = np.ascontiguousarray(count, dtype=np.int32)
    m = A.Microbatches(len(enc), ptr(_nonempty(enc), C.c_int64),
                       ptr(_nonempty(gen), C.c_int64),
                       ptr(_nonempty(count), C.c_int32))
    m._keep = (enc, gen, count)
    return m


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


# ----------------------------------------------------------------- planner
class CostModelHandle:
    def __init__(self, planner, model: Model, cluster: Cluster, book: Book):
        self.planner, self.model, self.cluster, self.book = planner, model, cluster, book
        rows = (A.ProfileRow * max(1, len(book.rows)))()
        for i, (mod, tp, load, fwd, bwd) in enumerate(book.rows):
            rows[i] = A.ProfileRow(mod, tp, int(bwd is not None), 0, load, fwd,
                                   0.0 if bwd is None else bwd)
        cb = A.CostBook(rows, len(book.rows), book.analytic_efficiency,
                        book.analytic_bwd_fwd_ratio)
        self._mc, self._cc = model.to_c(), cluster.to_c()
        h = C.c_void_p()
        planner._check(planner.lib.cost_model_create(planner.ctx, C.byref(self._mc),
                                                     C.byref(self._cc), C.byref(cb),
                                                     C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.planner.lib.cost_model_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Planner:
    def __init__(self, lib: A.Library, device: int = 0):
        self.lib = lib
        ctx = C.c_void_p()
        self._check(lib.context_create(device, C.byref(ctx)))
        self.ctx = ctx

    def close(self):
        if self.ctx:
            self.lib.context_destroy(self.ctx)
            self.ctx = None

    def _check(self, status):
        if status != 0:
            msg = self.lib.last_error().decode(errors="replace")
            raise _ERRORS.get(status, MmplanError)(msg)

    # ---- warning log (CostModel::set_warning_sink) ------------------------
    def warnings_enable(self, on: bool = True):
        """Start (and clear) or stop the context's warning log."""
        self._check(self.lib.warnings_enable(self.ctx, 1 if on else 0))

    def warnings(self) -> list:
        """The strings the reference's CostModel would have appended to its
        warning sink since warnings_enable, in the reference's order."""
        n = self.lib.warnings_count(self.ctx)
        return [self.lib.warning_at(self.ctx, i).decode() for i in range(n)]

    # ---- cost model ------------------------------------------------------
    def cost_model(self, model: Model, cluster: Cluster, book: Book) -> CostModelHandle:
        return CostModelHandle(self, model, cluster, book)

    def cost_sizes(self, batch: SampleBatch) -> np.ndarray:
        out = np.zeros(batch.n, dtype=np.int64)
        s = batch.to_c()
        self._check(self.lib.cost_sizes(self.ctx, C.byref(s), ptr(_nonempty(out), C.c_int64)))
        return out

    def unit_times(self, cm, module, tp, loads):
        loads = _f64(np.atleast_1d(loads))
        f = np.zeros_like(loads)
        b = np.zeros_like(loads)
        self._check(self.lib.unit_times(self.ctx, cm.h, module, tp, len(loads),
                                        ptr(loads, C.c_double), ptr(f, C.c_double),
                                        ptr(b, C.c_double)))
        return f, b

    def memory_check(self, cm, plan: PlanSpec):
        r = A.MemoryReport()
        pc = plan.to_c()
        self._check(self.lib.memory_check(self.ctx, cm.h, C.byref(pc), C.byref(r)))
        return r

    def build_stage_times(self, cm, plan: PlanSpec, enc, gen, count):
        mbs = microbatches_to_c(enc, gen, count)
        p = plan.virtual_stages()
        f = np.zeros((len(enc), p))
        b = np.zeros((len(enc), p))
        pc = plan.to_c()
        self._check(self.lib.build_stage_times(self.ctx, cm.h, C.byref(pc), C.byref(mbs),
                                               ptr(f, C.c_double), ptr(b, C.c_double)))
        return f, b

    def microbatch_fwd_keys(self, cm, plan: PlanSpec, enc, gen, count):
        mbs = microbatches_to_c(enc, gen, count)
        k = np.zeros(len(enc))
        pc = plan.to_c()
        self._check(self.lib.microbatch_fwd_keys(self.ctx, cm.h, C.byref(pc), C.byref(mbs),
                                                 ptr(_nonempty(k), C.c_double)))
        return k

    def compute_stats(self, batch: SampleBatch, seq_len: int):
        out = A.WorkloadStats()
        s = batch.to_c()
        self._check(self.lib.compute_stats(self.ctx, C.byref(s), seq_len, C.byref(out)))
        return out

    # ---- intra -----------------------------------------------------------
    def intra_partition(self, sizes, m, order=ASCENDING, equal_counts=False) -> IntraPartition:
        sizes = _f64(sizes)
        n = len(sizes)
        flat = np.zeros(max(n, 1), dtype=np.int32)
        offs = np.zeros(max(m, 0) + 1, dtype=np.int64)
        self._check(self.lib.intra_partition(self.ctx, ptr(_nonempty(sizes), C.c_double), n, m,
                                             order, int(equal_counts),
                                             ptr(flat, C.c_int32), ptr(offs, C.c_int64)))
        return IntraPartition([flat[offs[g]:offs[g + 1]].tolist() for g in range(m)])

    def intra_reorder_order(self, sizes, m, order=ASCENDING):
        return self.intra_partition(sizes, m, order).flat()

    def block_group_loads(self, sizes, order, m):
        sizes, order = _f64(sizes), _i32(order)
        out = np.zeros(m)
        self._check(self.lib.block_group_loads(self.ctx, ptr(_nonempty(sizes), C.c_double),
                                               ptr(_nonempty(order), C.c_int32), len(order), m,
                                               ptr(out, C.c_double)))
        return out

    def select_min(self, keys, pending, k):
        keys, pending = _f64(keys), _i32(pending)
        out = np.zeros(max(k, 1), dtype=np.int32)
        self._check(self.lib.select_min(self.ctx, ptr(_nonempty(keys), C.c_double), len(keys),
                                        ptr(_nonempty(pending), C.c_int32), len(pending), k,
                                        ptr(out, C.c_int32)))
        return out[:k].tolist()

    def select_closest(self, keys, pending, k, target):
        keys, pending = _f64(keys), _i32(pending)
        out = np.zeros(max(k, 1), dtype=np.int32)
        self._check(self.lib.select_closest(self.ctx, ptr(_nonempty(keys), C.c_double), len(keys),
                                            ptr(_nonempty(pending), C.c_int32), len(pending), k,
                                            float(target), ptr(out, C.c_int32)))
        return out[:k].tolist()

    # ---- simulator -------------------------------------------------------
    def schedule(self, fwd, bwd, vpp=1) -> Timeline:
        fwd, bwd = _f64(fwd), _f64(bwd)
        l, p = fwd.shape
        ne = 2 * l * p
        dev, mb, st, ph = (np.zeros(ne, dtype=np.int32) for _ in range(4))
        s, e = np.zeros(ne), np.zeros(ne)
        devices = p // vpp if vpp >= 1 and p % vpp == 0 else p
        busy = np.zeros(max(devices, 1))
        it = C.c_double()
        self._check(self.lib.schedule(self.ctx, ptr(fwd, C.c_double), ptr(bwd, C.c_double), l, p,
                                      vpp, ptr(dev, C.c_int32), ptr(mb, C.c_int32),
                                      ptr(st, C.c_int32), ptr(ph, C.c_int32), ptr(s, C.c_double),
                                      ptr(e, C.c_double), C.byref(it), ptr(busy, C.c_double)))
        return Timeline(dev, mb, st, ph, s, e, it.value, busy, devices, l, p)

    def schedule_1f1b(self, fwd, bwd) -> Timeline:
        return self.schedule(fwd, bwd, 1)

    def schedule_interleaved(self, fwd, bwd, vpp) -> Timeline:
        return self.schedule(fwd, bwd, vpp)

    def get_intervals(self, tl: Timeline):
        n = len(tl.start)
        cap = max(n, 1)
        ni = C.c_int64()
        s, e = np.zeros(cap), np.zeros(cap)
        fo = np.zeros(cap + 1, dtype=np.int64)
        fm = np.zeros(cap, dtype=np.int32)
        arr = [_i32(tl.device), _i32(tl.microbatch), _i32(tl.stage), _i32(tl.phase)]
        st, en = _f64(tl.start), _f64(tl.end)
        self._check(self.lib.get_intervals(self.ctx, n, *[ptr(_nonempty(a), C.c_int32) for a in arr],
                                           ptr(_nonempty(st), C.c_double),
                                           ptr(_nonempty(en), C.c_double), C.byref(ni),
                                           ptr(s, C.c_double), ptr(e, C.c_double),
                                           ptr(fo, C.c_int64), ptr(fm, C.c_int32)))
        k = ni.value
        return [Interval(float(s[i]), float(e[i]), fm[fo[i]:fo[i + 1]].tolist()) for i in range(k)]

    def interval_windows(self, fwd, bwd):
        fwd, bwd = _f64(fwd), _f64(bwd)
        l, p = fwd.shape
        out = np.zeros(l)
        self._check(self.lib.interval_windows(self.ctx, ptr(fwd, C.c_double), ptr(bwd, C.c_double),
                                              l, p, ptr(out, C.c_double)))
        return out

    def exhaustive_order(self, fwd, bwd, vpp=1, with_all=False):
        """Makespan of every ordering of the rows (tests/test_reorder.cpp:215-239):
        returns (best makespan, first order attaining it, all makespans in
        std::next_permutation order or None)."""
        fwd = np.ascontiguousarray(fwd, dtype=np.float64)
        bwd = np.ascontiguousarray(bwd, dtype=np.float64)
        l, p = fwd.shape
        best = C.c_double()
        order = np.zeros(l, dtype=np.int32)
        allt = np.zeros(math.factorial(l)) if with_all else None
        self._check(self.lib.exhaustive_order(self.ctx, ptr(fwd, C.c_double), ptr(bwd, C.c_double),
                                              l, p, vpp, C.byref(best), ptr(order, C.c_int32),
                                              ptr(allt, C.c_double)))
        return best.value, order.tolist(), allt

    def schedule_batch(self, fwd, bwd, vpp=1, with_busy=False):
        fwd, bwd = _f64(fwd), _f64(bwd)
        B, l, p = fwd.shape
        it = np.zeros(B)
        busy = np.zeros((B, p // vpp)) if with_busy else None
        self._check(self.lib.schedule_batch(self.ctx, B, ptr(fwd, C.c_double), ptr(bwd, C.c_double),
                                            l, p, vpp, ptr(it, C.c_double),
                                            ptr(busy, C.c_double)))
        return (it, busy) if with_busy else it

    def simulate_iteration(self, cm, plan: PlanSpec, groups):
        """groups: list of (enc[], gen[], count[]) per coupled group."""
        offs = np.zeros(len(groups) + 1, dtype=np.int64)
        enc, gen, cnt = [], [], []
        for g, (e, ge, c) in enumerate(groups):
            enc.extend(e), gen.extend(ge), cnt.extend(c)
            offs[g + 1] = len(enc)
        mbs = microbatches_to_c(enc, gen, cnt)
        t, st, bub = C.c_double(), C.c_double(), C.c_double()
        sg = C.c_int32()
        gt = np.zeros(max(1, len(groups)))
        pc = plan.to_c()
        self._check(self.lib.simulate_iteration(self.ctx, cm.h, C.byref(pc), len(groups),
                                                ptr(offs, C.c_int64), C.byref(mbs), C.byref(t),
                                                ptr(gt, C.c_double), C.byref(sg), C.byref(st),
                                                C.byref(bub)))
        return dict(t_iter=t.value, group_times=gt[:len(groups)], slowest_group=sg.value,
                    slowest_group_time=st.value, mean_bubble_fraction=bub.value)

    # ---- inter -----------------------------------------------------------
    def inter_reorder(self, fwd, bwd, keys, vpp=1):
        fwd, bwd, keys = _f64(fwd), _f64(bwd), _f64(keys)
        l, p = fwd.shape if fwd.ndim == 2 else (len(keys), 0)
        out = np.zeros(max(l, 1), dtype=np.int32)
        self._check(self.lib.inter_reorder(self.ctx, ptr(_nonempty(fwd.ravel()), C.c_double),
                                           ptr(_nonempty(bwd.ravel()), C.c_double), l, p,
                                           ptr(_nonempty(keys), C.c_double), vpp,
                                           ptr(out, C.c_int32)))
        return out[:l].tolist()

    def inter_reorder_batch(self, fwd, bwd, keys, vpp=1):
        fwd, bwd, keys = _f64(fwd), _f64(bwd), _f64(keys)
        B, l, p = fwd.shape
        out = np.zeros((B, l), dtype=np.int32)
        self._check(self.lib.inter_reorder_batch(self.ctx, B, ptr(fwd, C.c_double),
                                                 ptr(bwd, C.c_double), l, p,
                                                 ptr(keys, C.c_double), vpp, ptr(out, C.c_int32)))
        return out

    # ---- disaggregated ---------------------------------------------------
    @staticmethod
    def _mode(intra=True, inter=True, sort_order=ASCENDING):
        return A.ReorderMode(int(intra), int(inter), int(sort_order))

    def disaggregated_reorder(self, cm, plan: PlanSpec, batch: SampleBatch,
                              intra=True, inter=True, sort_order=ASCENDING) -> ReorderReport:
        n = batch.n
        dp = plan.backbone.dp
        order = np.zeros(max(n, 1), dtype=np.int32)
        lb, la = np.zeros(max(dp, 1)), np.zeros(max(dp, 1))
        rep = A.ReorderReport(ptr(order, C.c_int32), ptr(lb, C.c_double), ptr(la, C.c_double), 0.0, 0.0)
        s = batch.to_c()
        pc = plan.to_c()
        md = self._mode(intra, inter, sort_order)
        self._check(self.lib.disaggregated_reorder(self.ctx, cm.h, C.byref(pc), C.byref(md),
                                                   C.byref(s), C.byref(rep)))
        return ReorderReport(order[:n].copy(), lb[:dp].copy(), la[:dp].copy(),
                             rep.t_iter_before, rep.t_iter_after)

    def reorder_stream(self, cm, plan: PlanSpec, samples: SampleBatch, n_batches,
                       intra=True, inter=True, sort_order=ASCENDING, with_kept=False):
        n = samples.n
        dp = plan.backbone.dp
        order = np.zeros(n, dtype=np.int32)
        lb, la = np.zeros(n_batches * dp), np.zeros(n_batches * dp)
        tb, ta = np.zeros(n_batches), np.zeros(n_batches)
        kept = np.zeros(n_batches, dtype=np.uint8) if with_kept else None
        s = samples.to_c()
        pc = plan.to_c()
        md = self._mode(intra, inter, sort_order)
        self._check(self.lib.reorder_stream(self.ctx, cm.h, C.byref(pc), C.byref(md), C.byref(s),
                                            n_batches, ptr(order, C.c_int32), ptr(lb, C.c_double),
                                            ptr(la, C.c_double), ptr(tb, C.c_double),
                                            ptr(ta, C.c_double), ptr(kept, C.c_uint8)))
        out = dict(output_order=order, load_before=lb.reshape(n_batches, dp),
                   load_after=la.reshape(n_batches, dp), t_iter_before=tb, t_iter_after=ta)
        if with_kept:
            out["greedy_kept"] = kept
        return out

    # ---- orchestration ---------------------------------------------------
    def predict_times(self, cm, stats: A.WorkloadStats, plans):
        plans = list(plans)
        arr = (A.Plan * len(plans))(*[p.to_c() for p in plans])
        out = (A.PredictedTimes * len(plans))()
        self._check(self.lib.predict_times(self.ctx, cm.h, C.byref(stats), arr, len(plans), out))
        return [(o.t_warm, o.t_steady, o.t_iter) for o in out]

    def enumerate_parallelism(self, cluster: Cluster, global_batch):
        cnt = C.c_int64()
        cc = cluster.to_c()
        self._check(self.lib.enumerate_parallelism(self.ctx, C.byref(cc), global_batch,
                                                   C.byref(cnt), None, 0))
        buf = (A.Tuple * max(1, cnt.value))()
        self._check(self.lib.enumerate_parallelism(self.ctx, C.byref(cc), global_batch,
                                                   C.byref(cnt), buf, cnt.value))
        return [(t.tp_me, t.dp_me, t.tp_lm, t.dp_lm, t.tp_mg, t.dp_mg)
                for t in buf[:cnt.value]]

    def solve_subproblem(self, cm, stats, tuples, global_batch, vpp=1):
        tuples = list(tuples)
        arr = (A.Tuple * max(1, len(tuples)))(*[tuple_to_c(t) for t in tuples])
        out = (A.Candidate * max(1, len(tuples)))()
        self._check(self.lib.solve_subproblem(self.ctx, cm.h, C.byref(stats), arr, len(tuples),
                                              global_batch, vpp, out))
        return [Candidate.from_c(c) for c in out[:len(tuples)]]

    def brute_force_oracle(self, cm, stats, global_batch, vpp=1, gpu_cap=32):
        """brute_force_oracle (src/orchestrator.cpp:433-491)."""
        res = A.OrchestrationResult()
        self._check(self.lib.brute_force_oracle(self.ctx, cm.h, C.byref(stats), global_batch, vpp,
                                                gpu_cap, C.byref(res)))
        return dict(best=PlanSpec.from_c(res.best),
                    times=(res.times.t_warm, res.times.t_steady, res.times.t_iter),
                    candidates_evaluated=res.candidates_evaluated)

    # ---- multi-GPU reorder stream (one process per GPU) ------------------
    def peer_buffer_create(self, n_samples: int):
        """Replica buffer of the whole ordering on this planner's GPU:
        (device pointer, 64-byte IPC handle)."""
        p, h = C.c_void_p(), A.PeerHandle()
        self._check(self.lib.peer_buffer_create(self.ctx, n_samples, C.byref(p), C.byref(h)))
        return p.value, bytes(h.bytes)

    def peer_buffer_destroy(self, replica: int):
        self._check(self.lib.peer_buffer_destroy(self.ctx, C.c_void_p(replica)))

    def peer_group_open(self, rank: int, world: int, replica: int, n_samples: int, handles):
        arr = (A.PeerHandle * world)()
        for i, h in enumerate(handles):
            C.memmove(arr[i].bytes, h, 64)
        g = C.c_void_p()
        self._check(self.lib.peer_group_open(self.ctx, rank, world, C.c_void_p(replica), n_samples,
                                             arr, C.byref(g)))
        return g

    def peer_group_close(self, group):
        self._check(self.lib.peer_group_close(group))

    def shard_range(self, n_batches: int, rank: int, world: int):
        f, c = C.c_int64(), C.c_int64()
        self._check(self.lib.shard_range(n_batches, rank, world, C.byref(f), C.byref(c)))
        return f.value, c.value

    def ingest_trace(self, data: bytes, seq_len_cap: int) -> "SampleBatch":
        """ingest_trace (src/workload.cpp:115-153): JSONL bytes -> SampleBatch.
        Raises TraceError with kind()/line() like the reference."""
        res = A.TraceResult()
        st = self.lib.ingest_trace(self.ctx, data, len(data), seq_len_cap, None, C.byref(res))
        self._trace_check(st, res)
        n, ni, na = res.n_samples, res.n_image, res.n_audio
        out = SampleBatch(np.zeros(n, np.int32), np.zeros(n + 1, np.int32),
                          np.zeros(max(ni, 1), np.int32), np.zeros(n + 1, np.int32),
                          np.zeros(max(na, 1), np.int32))
        csr = A.TraceCsr(n, ni, na, out.text.ctypes.data, out.image_offsets.ctypes.data,
                         out.image_tokens.ctypes.data, out.audio_offsets.ctypes.data,
                         out.audio_tokens.ctypes.data)
        st = self.lib.ingest_trace(self.ctx, data, len(data), seq_len_cap, C.byref(csr),
                                   C.byref(res))
        self._trace_check(st, res)
        out.image_tokens = out.image_tokens[:ni]
        out.audio_tokens = out.audio_tokens[:na]
        return out

    def ingest_trace_dev(self, data_ptr: int, length: int, seq_len_cap: int, out=None):
        """dtb_ingest_trace_dev: device bytes -> device CSR.  out: None (sizes
        only) or dict(cap_samples, cap_image, cap_audio, text_tokens,
        image_offsets, image_tokens, audio_offsets, audio_tokens) of device
        pointers.  Returns the TraceResult."""
        res = A.TraceResult()
        csr = None
        if out is not None:
            csr = A.TraceCsr(out["cap_samples"], out["cap_image"], out["cap_audio"],
                             out["text_tokens"], out["image_offsets"], out["image_tokens"],
                             out["audio_offsets"], out["audio_tokens"])
        st = self.lib.ingest_trace_dev(self.ctx, data_ptr, length, seq_len_cap,
                                       C.byref(csr) if csr is not None else None, C.byref(res))
        self._trace_check(st, res)
        return res

    def _trace_check(self, status, res):
        if status == 9:
            msg = self.lib.last_error().decode(errors="replace")
            kind = "ParseError" if res.error_kind == 1 else "InvariantViolation"
            raise TraceError(msg, kind, res.error_line)
        self._check(status)

    def rigid_baseline(self, cm, stats, global_batch, vpp=1):
        """rigid_baseline (src/orchestrator.cpp:407-431)."""
        plan = A.Plan()
        self._check(self.lib.rigid_baseline(self.ctx, cm.h, C.byref(stats), global_batch, vpp,
                                            C.byref(plan)))
        return PlanSpec.from_c(plan)

    def model_orchestration(self, cm, stats, global_batch, vpp=1, keep_candidates=False):
        res = A.OrchestrationResult()
        cands, cap = None, 0
        if keep_candidates:
            cap = len(self.enumerate_parallelism(cm.cluster, global_batch))
            cands = (A.Candidate * max(1, cap))()
        self._check(self.lib.model_orchestration(self.ctx, cm.h, C.byref(stats), global_batch, vpp,
                                                 C.byref(res), cands, cap))
        out = dict(best=PlanSpec.from_c(res.best),
                   times=(res.times.t_warm, res.times.t_steady, res.times.t_iter),
                   candidates_evaluated=res.candidates_evaluated,
                   solve_seconds=res.solve_seconds)
        if keep_candidates:
            out["candidates"] = [Candidate.from_c(c) for c in cands[:cap]]
        return out
