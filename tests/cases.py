"""Synthetic step inputs shared by the parity tests (seeded, small)."""
from __future__ import annotations

import numpy as np


def zipf_ids(rng, rows, n, s=1.05):
    """Zipf-skewed ids in [0, rows): rank k has mass ~ (k+1)^-s (low ids hot,
    like the reference DataGenerator, data.cpp:85-98,128-136)."""
    k = np.arange(1, rows + 1, dtype=np.float64)
    p = k ** (-s)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    u = rng.random(n)
    return np.minimum(np.searchsorted(cdf, u, side="right"), rows - 1).astype(np.uint32)


def make_batch(rng, rows, B, max_len=6, zipf=1.05, min_len=0, fixed_len=None):
    """One rank's batch: sample-major lengths [B*F] and concatenated ids."""
    F = len(rows)
    if fixed_len is not None:
        lengths = np.full(B * F, fixed_len, np.uint32)
    else:
        lengths = rng.integers(min_len, max_len + 1, size=B * F).astype(np.uint32)
    ids = []
    for b in range(B * F):
        f = b % F
        ids.append(zipf_ids(rng, int(rows[f]), int(lengths[b]), zipf))
    ids = np.concatenate(ids) if ids else np.zeros(0, np.uint32)
    return lengths, ids.astype(np.uint32)


def upstream(rng, B, sum_dims, scale=1e-3):
    return (scale * rng.standard_normal((B, sum_dims))).astype(np.float32)
