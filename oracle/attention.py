"""Numpy restatement of the reference HSTU attention operator (TEST ORACLE).

Follows ``/root/reference/pkg/src/jaggedcp/attention.py``:

* ``silu``/``sigmoid``      -> attention.py:56-75 (sign-split stable forms)
* ``bucketize_array``       -> attention.py:83-86 (f64 log1p, floor, clip)
* ``compute_bias``          -> attention.py:89-94
* ``hstu_fwd_seq``          -> attention.py:135-147 (one sequence, one head)
* ``blockwise_partial``     -> attention.py:151-184
* ``hstu_bwd_seq``          -> attention.py:207-228 (analytic backward)
* ``normal_init_ts_weights``-> attention.py:43-47

Multi-head (``num_heads > 1``) is the per-head composition of the pinned
single-head operator on column blocks ``values[:, h*d:(h+1)*d]`` with the
scale ``sqrt(d)`` of one head; the bias (and so ``d_ts_weights``) is shared by
all heads.  The optional positional bias ``pos_weights[min(i-j, P-1)]`` is an
opt-in extension (off by default; parity unpinned).
"""

from __future__ import annotations

import math

import numpy as np


def silu(x):
    """attention.py:56-66."""
    xv = np.asarray(x)
    if not np.issubdtype(xv.dtype, np.floating):
        xv = xv.astype(np.float64)
    out = np.empty_like(xv)
    pos = xv >= 0
    out[pos] = xv[pos] / (1.0 + np.exp(-xv[pos]))
    e = np.exp(xv[~pos])
    out[~pos] = xv[~pos] * e / (1.0 + e)
    return out if out.ndim else out[()]


def sigmoid(x: np.ndarray) -> np.ndarray:
    """attention.py:69-75."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def bucketize_array(deltas: np.ndarray, num_buckets: int) -> np.ndarray:
    """attention.py:83-86: min(nb-1, floor(log1p(max(delta, 0)))) via f64."""
    clipped = np.maximum(np.asarray(deltas).astype(np.float64), 0.0)
    idx = np.floor(np.log1p(clipped)).astype(np.int64)
    return np.clip(idx, 0, num_buckets - 1)


def bucketize(delta: int, num_buckets: int) -> int:
    """attention.py:78-80."""
    return int(bucketize_array(np.asarray([delta], dtype=np.int64), num_buckets)[0])


def compute_bias(ts_q, ts_k, ts_weights, num_buckets: int) -> np.ndarray:
    """attention.py:89-94: |q| x |k| weights picked by pairwise deltas."""
    tq = np.asarray(ts_q, dtype=np.int64)
    tk = np.asarray(ts_k, dtype=np.int64)
    return np.asarray(ts_weights, dtype=np.float64)[bucketize_array(tq[:, None] - tk[None, :], num_buckets)]


def _pos_bias(lq: int, lk: int, q_pos0: int, k_pos0: int, pos_weights, dt) -> np.ndarray:
    """Extension (default off): pos_weights[clip(i - j, 0, P-1)]."""
    pw = np.asarray(pos_weights, dtype=np.float64)
    i = np.arange(q_pos0, q_pos0 + lq)[:, None]
    j = np.arange(k_pos0, k_pos0 + lk)[None, :]
    return pw[np.clip(i - j, 0, pw.size - 1)].astype(dt)


def normal_init_ts_weights(num_buckets: int, seed: int, mean: float = 0.0, stddev: float = 0.02) -> np.ndarray:
    """attention.py:43-47 (BiasParams.normal_init)."""
    rng = np.random.default_rng(seed)
    return rng.normal(mean, stddev, size=num_buckets).astype(np.float64)


def hstu_fwd_seq(qb, kb, vb, tb, ts_weights, num_buckets, pos_weights=None):
    """attention.py:140-147 for one sequence and one head (dtype of qb)."""
    dt = qb.dtype
    L = qb.shape[0]
    scale = dt.type(math.sqrt(qb.shape[1]))
    bias = compute_bias(tb, tb, ts_weights, num_buckets).astype(dt)
    if pos_weights is not None:
        bias = bias + _pos_bias(L, L, 0, 0, pos_weights, dt)
    scores = (qb @ kb.T + bias) / scale
    gated = silu(scores)
    keep = np.tril(np.ones((L, L), dtype=bool))
    return np.where(keep, gated, dt.type(0)) @ vb


def hstu_bwd_seq(qb, kb, vb, tb, g, ts_weights, num_buckets, pos_weights=None):
    """attention.py:212-228 for one sequence and one head.

    Returns (dq, dk, dv, d_w[nb] f64, d_pos[P] f64 or None)."""
    dt = qb.dtype
    L = qb.shape[0]
    scale = dt.type(math.sqrt(qb.shape[1]))
    buckets = bucketize_array(tb[:, None] - tb[None, :], num_buckets)
    bias = np.asarray(ts_weights, dtype=np.float64)[buckets].astype(dt)
    if pos_weights is not None:
        bias = bias + _pos_bias(L, L, 0, 0, pos_weights, dt)
    scores = (qb @ kb.T + bias) / scale
    sig = sigmoid(scores)
    keep = np.tril(np.ones((L, L), dtype=bool))
    gated = np.where(keep, scores * sig, dt.type(0))
    dv = gated.T @ g
    d_gated = g @ vb.T
    d_scores = np.where(keep, d_gated * sig * (1.0 + scores * (1.0 - sig)), dt.type(0))
    dq = (d_scores @ kb) / scale
    dk = (d_scores.T @ qb) / scale
    d_bias = (d_scores / scale).astype(np.float64)
    d_w = np.bincount(buckets.ravel(), weights=d_bias.ravel(), minlength=num_buckets)
    d_pos = None
    if pos_weights is not None:
        P = int(np.asarray(pos_weights).size)
        rel = np.clip(np.arange(L)[:, None] - np.arange(L)[None, :], 0, P - 1)
        d_pos = np.bincount(rel.ravel(), weights=d_bias.ravel(), minlength=P)
    return dq, dk, dv, d_w, d_pos


def _heads(values: np.ndarray, num_heads: int):
    D = values.shape[1]
    if D % num_heads:
        raise ValueError(f"embed_dim {D} not divisible by num_heads {num_heads}")
    d = D // num_heads
    return d, [(h * d, (h + 1) * d) for h in range(num_heads)]


def hstu_forward(q, k, v, ts, offsets, ts_weights, num_buckets=16, num_heads=1, pos_weights=None):
    """attention.py:125-148 over a jagged batch; multi-head = per-head loop."""
    offsets = np.asarray(offsets, dtype=np.int64)
    out = np.zeros_like(v)
    _, cols = _heads(q, num_heads)
    for b in range(len(offsets) - 1):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        if hi == lo:
            continue
        for c0, c1 in cols:
            out[lo:hi, c0:c1] = hstu_fwd_seq(
                q[lo:hi, c0:c1], k[lo:hi, c0:c1], v[lo:hi, c0:c1], ts[lo:hi], ts_weights, num_buckets, pos_weights
            )
    return out


def hstu_backward(q, k, v, ts, offsets, g, ts_weights, num_buckets=16, num_heads=1, pos_weights=None):
    """attention.py:187-234 over a jagged batch; d_w summed over heads."""
    offsets = np.asarray(offsets, dtype=np.int64)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    d_w = np.zeros(num_buckets, dtype=np.float64)
    d_pos = None if pos_weights is None else np.zeros(np.asarray(pos_weights).size, dtype=np.float64)
    _, cols = _heads(q, num_heads)
    for b in range(len(offsets) - 1):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        if hi == lo:
            continue
        for c0, c1 in cols:
            a, bb, c, w, p = hstu_bwd_seq(
                q[lo:hi, c0:c1], k[lo:hi, c0:c1], v[lo:hi, c0:c1], ts[lo:hi], g[lo:hi, c0:c1],
                ts_weights, num_buckets, pos_weights,
            )
            dq[lo:hi, c0:c1] = a
            dk[lo:hi, c0:c1] = bb
            dv[lo:hi, c0:c1] = c
            d_w += w
            if p is not None:
                d_pos += p
    return dq, dk, dv, d_w, d_pos


def blockwise_partial(q, q_seq_ids, q_positions, ts_q, k, k_seq_ids, k_positions, ts_k, v,
                      ts_weights, num_buckets=16):
    """attention.py:151-184 (single head): masked partial over one K/V block."""
    if k.shape[0] != v.shape[0]:
        raise ValueError(f"k has {k.shape[0]} rows but v has {v.shape[0]}")
    dt = q.dtype
    if q.shape[0] == 0 or k.shape[0] == 0:
        return np.zeros((q.shape[0], v.shape[1] if v.ndim == 2 else 0), dtype=dt)
    scale = dt.type(math.sqrt(q.shape[1]))
    bias = compute_bias(ts_q, ts_k, ts_weights, num_buckets).astype(dt)
    scores = (q @ k.T + bias) / scale
    gated = silu(scores)
    allowed = (np.asarray(q_seq_ids)[:, None] == np.asarray(k_seq_ids)[None, :]) & (
        np.asarray(k_positions)[None, :] <= np.asarray(q_positions)[:, None]
    )
    return np.where(allowed, gated, dt.type(0)) @ v
