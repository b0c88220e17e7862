"""Fixtures mirroring the reference's test support
(proj/tests/support/fixtures.hpp:27-86, configs.hpp:26-135) plus the
BASELINE.json configurations.  Pure data: no oracle, no device."""
from __future__ import annotations

import numpy as np

from paper_2408_04275_b200.api import (ALLOWED_TP, BACKBONE, ENCODER, GENERATOR, Book,
                                       Choice, Cluster, Model, Module, PlanSpec)

GiB = float(1 << 30)


def toy_model() -> Model:  # fixtures.hpp:27-37
    return Model(
        encoder=Module(8, 512, 2048, 8, 8, 1e9, 2e9, 1e8),
        backbone=Module(16, 1024, 4096, 16, 16, 8e9, 16e9, 2e8),
        generator=Module(8, 640, 2560, 10, 10, 2e9, 4e9, 1e8),
        seq_len=8192)


def toy_cluster(gpus: int) -> Cluster:  # fixtures.hpp:39-48
    return Cluster(gpus, 8, 312e12, 80e9, 300e9, 100e9)


def quiet_cluster(gpus: int) -> Cluster:  # test_orchestrator.cpp:38-43
    c = toy_cluster(gpus)
    c.intra_node_bw = c.inter_node_bw = 1e30
    return c


def flat_book(enc, lm, gen) -> Book:  # fixtures.hpp:58-66
    b = Book()
    for tp in ALLOWED_TP:
        b.add_row(ENCODER, tp, 0, enc, 2 * enc)
        b.add_row(BACKBONE, tp, 0, lm, 2 * lm)
        b.add_row(GENERATOR, tp, 0, gen, 2 * gen)
    return b


def tp_scaled_book(enc, lm, gen, eff=0.85) -> Book:  # fixtures.hpp:68-84
    b = Book()
    for tp in ALLOWED_TP:
        speedup = 1.0
        k = 1
        while k < tp:
            speedup *= 2.0 * eff
            k *= 2
        b.add_row(ENCODER, tp, 0, enc / speedup, 2 * enc / speedup)
        b.add_row(BACKBONE, tp, 0, lm / speedup, 2 * lm / speedup)
        b.add_row(GENERATOR, tp, 0, gen / speedup, 2 * gen / speedup)
    return b


def desk_book(rows=(("encoder", 0.110, 0.004), ("backbone", 0.760, 0.760),
                    ("generator", 0.420, 0.008))) -> Book:
    """configs.hpp:79-102: 2 load rows per TP, 1.8x per TP doubling.  The
    reference writes the CSV with std::to_string (6 decimals) and parses it
    back, so values are rounded the same way here."""
    b = Book()
    idx = {"encoder": ENCODER, "backbone": BACKBONE, "generator": GENERATOR}
    for name, base, floor in rows:
        for tp in ALLOWED_TP:
            speedup = 1.0
            k = 1
            while k < tp:
                speedup *= 1.8
                k *= 2
            for load in (0.0, 8192.0):
                fwd = (floor + (base - floor) * load / 8192.0) / speedup
                f6 = float("%.6f" % fwd)
                b6 = float("%.6f" % (2.0 * fwd))
                b.add_row(idx[name], tp, load, f6, b6)
    return b


def desk_model() -> Model:  # configs.hpp:55-77
    return Model(
        encoder=Module(32, 1280, 5120, 16, 16, 3.4 * GiB, 10 * GiB, 0.25 * GiB),
        backbone=Module(32, 4096, 11008, 32, 32, 26 * GiB, 78 * GiB, 2 * GiB),
        generator=Module(32, 1280, 5120, 16, 16, 4 * GiB, 12 * GiB, 0.25 * GiB),
        seq_len=8192, frozen_backward_factor=0.3333333333333333)


def desk_cluster(gpus: int) -> Cluster:  # configs.hpp:104-114
    return Cluster(gpus, 8, 312e12, 80 * GiB, 150e9, 25e9)


def a800_cluster(gpus: int) -> Cluster:
    return Cluster(gpus, 8, 312e12, 80e9, 150e9, 100e9)


def mllm72b_model() -> Model:
    """BASELINE config 3: Llama3-70B backbone + ViT-H encoder + SD2.1-sized
    generator; memory P = 6 B/param, S = 12 B/param."""
    def mod(layers, hidden, ffn, heads, groups, act):
        m = Module(layers, hidden, ffn, heads, groups)
        params = layers * (hidden * hidden * (2.0 + 2.0 * groups / heads) + 3.0 * hidden * ffn)
        m.param_grad_bytes, m.optimizer_bytes, m.activation_bytes_per_mb = 6 * params, 12 * params, act
        return m
    return Model(encoder=mod(32, 1280, 5120, 16, 16, 0.25 * GiB),
                 backbone=mod(80, 8192, 28672, 64, 8, 4 * GiB),
                 generator=mod(28, 1536, 6144, 24, 24, 0.5 * GiB),
                 seq_len=8192, frozen_backward_factor=1.0 / 3.0)


def mllm72b_book() -> Book:
    return desk_book((("encoder", 0.110, 0.004), ("backbone", 6.1, 6.1),
                      ("generator", 0.520, 0.010)))


def llava_model() -> Model:
    """BASELINE config 2: ViT-L encoder {24,1024,4096,16} + Llama-7B backbone
    {32,4096,11008,32,32} and a near-zero-cost generator (the
    reference requires one, src/validate.cpp:59-62)."""
    return Model(encoder=Module(24, 1024, 4096, 16, 16, 1.2 * GiB, 3.6 * GiB, 0.2 * GiB),
                 backbone=Module(32, 4096, 11008, 32, 32, 26 * GiB, 78 * GiB, 2 * GiB),
                 generator=Module(1, 64, 256, 1, 1, 1e6, 1e6, 1e6),
                 seq_len=8192)


def llava_book() -> Book:
    return desk_book((("encoder", 0.090, 0.004), ("backbone", 0.760, 0.760),
                      ("generator", 0.0011, 0.0010)))


def plan(enc, lm, gen, bs, vpp=1) -> PlanSpec:
    return PlanSpec(Choice(*enc), Choice(*lm), Choice(*gen), bs, vpp)


def random_times(rng: np.random.Generator, l, p, lo=0.1, hi=2.0):
    """oracles.hpp:190-202 (numpy stream instead of mt19937_64)."""
    return rng.uniform(lo, hi, (l, p)), rng.uniform(lo, hi, (l, p))


def skewed_times(enc, p, base):  # test_reorder.cpp:35-46
    l = len(enc)
    f = np.full((l, p), float(base))
    f[:, 0] += np.asarray(enc, dtype=float)
    return f, 2.0 * f
