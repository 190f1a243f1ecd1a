"""Numpy restatement of the reference synthetic-input generator and error
metric (TEST ORACLE).

Follows ``/root/reference/pkg/src/jaggedcp/harness.py``:

* ``gen_synthetic_batch`` -> harness.py:116-145 (same RNG stream:
  ``default_rng([seed, rank])``; lengths, q, k, v, starts, gaps in order)
* ``bias seed``           -> harness.py:148-152 (``seed + 0x5EED``)
* ``concat_batches``      -> harness.py:155-168
* ``output_errors``       -> harness.py:189-206 (max abs, row-normalized)
"""

from __future__ import annotations

import numpy as np

MAX_TS_GAP_SECONDS = 1_000_000
BIAS_SEED_OFFSET = 0x5EED


def draw_lengths(rng, batch_size, length_dist="uniform", min_len=1, max_len=32,
                 lognorm_mu=3.0, lognorm_sigma=0.8, max_length=128):
    """harness.py:116-120."""
    if length_dist == "uniform":
        return rng.integers(min_len, max_len + 1, size=batch_size)
    raw = np.floor(rng.lognormal(lognorm_mu, lognorm_sigma, size=batch_size))
    return np.clip(raw, 1, max_length).astype(np.int64)


def gen_synthetic_batch(seed, rank, batch_size, embed_dim, dtype=np.float32, length_dist="uniform",
                        min_len=1, max_len=32, lognorm_mu=3.0, lognorm_sigma=0.8, max_length=128):
    """harness.py:123-145.  Returns dict(q, k, v, ts, offsets)."""
    rng = np.random.default_rng([seed, rank])
    seq_lengths = draw_lengths(rng, batch_size, length_dist, min_len, max_len, lognorm_mu, lognorm_sigma, max_length)
    offsets = np.concatenate([[0], np.cumsum(seq_lengths)]).astype(np.int64)
    total = int(offsets[-1])
    dt = np.dtype(dtype)
    q = rng.standard_normal((total, embed_dim), dtype=dt)
    k = rng.standard_normal((total, embed_dim), dtype=dt)
    v = rng.standard_normal((total, embed_dim), dtype=dt)
    starts = rng.integers(0, 1_000_000_000, size=batch_size)
    gaps = rng.integers(1, MAX_TS_GAP_SECONDS + 1, size=total)
    ts = np.zeros(total, dtype=np.int64)
    for b in range(batch_size):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        ts[lo:hi] = starts[b] + np.cumsum(gaps[lo:hi])
    return {"q": q, "k": k, "v": v, "ts": ts, "offsets": offsets}


def concat_batches(batches):
    """harness.py:155-168 (sequences in rank order)."""
    offs = [0]
    for b in batches:
        base = offs[-1]
        offs.extend(int(base + o) for o in b["offsets"][1:])
    return {
        "q": np.concatenate([b["q"] for b in batches]),
        "k": np.concatenate([b["k"] for b in batches]),
        "v": np.concatenate([b["v"] for b in batches]),
        "ts": np.concatenate([b["ts"] for b in batches]),
        "offsets": np.asarray(offs, dtype=np.int64),
    }


def output_errors(got, want):
    """harness.py:189-206: (max abs error, max row-normalized error)."""
    max_abs = 0.0
    max_rel = 0.0
    for g, w in zip(got, want):
        g = np.asarray(g, dtype=np.float64)
        w = np.asarray(w, dtype=np.float64)
        if g.shape[0] == 0:
            continue
        diff = np.abs(g - w)
        ref = np.abs(w)
        max_abs = max(max_abs, float(diff.max()))
        row_err = diff.max(axis=1) / np.maximum(1.0, ref.max(axis=1))
        max_rel = max(max_rel, float(row_err.max()))
    return max_abs, max_rel
