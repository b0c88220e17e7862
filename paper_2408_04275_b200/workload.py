"""Synthetic sample streams in the CSR layout of `dtb_samples`.

The reference's `synth_batch` (src/workload.cpp:33-113) draws with libm
(`std::log/exp/cos`) and std::mt19937_64, which is not reproducible on the
device (SURVEY.md §7 hard part 7).  Streams here are generated once on the
host with numpy's PCG64 and the SAME int32 arrays are fed to the GPU path and
to the CPU oracle, so parity never depends on the generator.

Two families:
  * skewed  — the reference's canonical skewed workload
    (proj/tests/support/configs.hpp:116-125): text lognormal(600, 0.8),
    image-subsequence tokens lognormal(1024, 0.47), image count
    geometric(mean 2), packed into seq_len with truncation in the order of
    src/workload.cpp:93-111.
  * mixed   — BASELINE config 4: the skewed text/count law, variable image
    resolution mapped to (res/16)^2 patch tokens from a fixed
    resolution set, and an audio clip (lognormal(750, 0.6) tokens) on 25% of
    samples, placed in `audio_subseqs` after the images.
  * dense   — the mixed family with at least one image per sample (no
    text-only samples): the equal-count greedy split then balances better
    than the incoming order and is KEPT on most batches, which exercises the
    permutation half of the intra path.
"""
from __future__ import annotations

import numpy as np

from .api import SampleBatch

RESOLUTIONS = np.array([224, 336, 448, 512, 672, 896])


def _lognormal_tokens(rng, median, sigma, size):
    v = np.rint(median * np.exp(sigma * rng.standard_normal(size)))
    return np.maximum(v, 1).astype(np.int64)


def synth_stream(n: int, seed: int = 1, family: str = "mixed",
                 seq_len: int = 8192) -> SampleBatch:
    """n samples of the given family as one CSR SampleBatch."""
    rng = np.random.Generator(np.random.PCG64(seed))
    text = np.clip(_lognormal_tokens(rng, 600.0, 0.8, n), 1, seq_len)
    budget = seq_len - text
    q = 1.0 / (1.0 + 2.0)  # geometric with mean 2 (src/workload.cpp:55-60)
    u = 1.0 - rng.random(n)  # (0, 1]
    count = np.floor(np.log(u) / np.log(1.0 - q)).astype(np.int64)
    count = np.minimum(count, 64)
    if family == "dense":
        count = np.maximum(count, 1)
    total = int(count.sum())
    if family == "skewed":
        draws = _lognormal_tokens(rng, 1024.0, 0.47, total)
    elif family in ("mixed", "dense"):
        draws = (RESOLUTIONS[rng.integers(0, len(RESOLUTIONS), total)] // 16) ** 2
    else:
        raise ValueError(family)
    owner = np.repeat(np.arange(n), count)
    # Truncate each sample's images to its remaining budget, in order
    # (min(budget, draw); stop adding once the budget is exhausted).
    start = np.concatenate([[0], np.cumsum(count)[:-1]])
    excl = np.cumsum(draws) - draws
    before = excl - excl[start[owner]] if total else excl
    tokens = np.minimum(draws, budget[owner] - before)
    keep = tokens > 0
    img_tokens = tokens[keep].astype(np.int32)
    img_counts = np.bincount(owner[keep], minlength=n)
    img_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(img_counts, out=img_off[1:])
    used = budget - np.bincount(owner[keep], weights=tokens[keep], minlength=n).astype(np.int64)
    if family in ("mixed", "dense"):
        has_audio = rng.random(n) < 0.25
        atok = _lognormal_tokens(rng, 750.0, 0.6, n)
        atok = np.minimum(atok, used)
        has_audio &= atok > 0
        aud_tokens = atok[has_audio].astype(np.int32)
        aud_off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(has_audio.astype(np.int64), out=aud_off[1:])
    else:
        aud_tokens = np.zeros(0, dtype=np.int32)
        aud_off = np.zeros(n + 1, dtype=np.int64)
    if img_off[-1] >= 2**31 or aud_off[-1] >= 2**31:
        raise ValueError("stream exceeds the int32 CSR offset limit")
    return SampleBatch(text.astype(np.int32), img_off.astype(np.int32), img_tokens,
                       aud_off.astype(np.int32), aud_tokens)


def write_trace(batch: SampleBatch) -> bytes:
    """write_trace (src/workload.cpp:157-165) of a SampleBatch: one nlohmann
    ordered_json dump per line — compact separators, keys text_tokens,
    image_subseqs, then audio_subseqs only when non-empty."""
    import json
    io, it = batch.image_offsets, batch.image_tokens
    ao, at = batch.audio_offsets, batch.audio_tokens
    text = batch.text.tolist()
    lines = []
    for i in range(batch.n):
        rec = {"text_tokens": text[i], "image_subseqs": it[io[i]:io[i + 1]].tolist()}
        if ao[i + 1] > ao[i]:
            rec["audio_subseqs"] = at[ao[i]:ao[i + 1]].tolist()
        lines.append(json.dumps(rec, separators=(",", ":")))
    return ("\n".join(lines) + "\n").encode()
