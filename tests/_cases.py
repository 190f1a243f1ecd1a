"""Seeded jagged inputs shared by the GPU parity tests (bf16-rounded, with
the matching f32 numpy copies the oracle consumes)."""

import numpy as np

import oracle
from oracle import harness as oh


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def make_case(lens, D, seed=0, nb=16, ts_gap_max=1_000_000, unsorted_ts=False):
    rng = np.random.default_rng(seed)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    q, k, v, g = (bf16_round(rng.standard_normal((T, D)).astype(np.float32)) for _ in range(4))
    ts = np.zeros(T, dtype=np.int64)
    for b, L in enumerate(lens):
        lo = int(offs[b])
        if unsorted_ts:
            ts[lo:lo + L] = rng.integers(0, 10**7, size=L)
        else:
            ts[lo:lo + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, ts_gap_max + 1, size=L))
    w = oracle.normal_init_ts_weights(nb, seed + 0x5EED)
    return dict(q=q, k=k, v=v, g=g, ts=ts, offsets=offs, w=w, nb=nb)


def synthetic(seed, rank, batch, max_len, H, d, dist="uniform", min_len=1):
    """Reference generator (harness.py:123) at embed_dim H*d, rounded to bf16."""
    b = oh.gen_synthetic_batch(seed, rank, batch, H * d, np.float32, dist, min_len, max_len,
                               float(np.log(1024)), 1.0, max(max_len, 8192))
    for key in ("q", "k", "v"):
        b[key] = bf16_round(b[key])
    return b


def to_cuda(case):
    import torch
    dev = "cuda"
    out = {}
    for key in ("q", "k", "v", "g"):
        if key in case:
            out[key] = torch.from_numpy(case[key]).to(dev).bfloat16()
    out["ts"] = torch.from_numpy(case["ts"]).to(dev)
    out["offsets"] = torch.from_numpy(case["offsets"]).to(dev)
    out["w"] = torch.from_numpy(np.asarray(case["w"], dtype=np.float32)).to(dev)
    return out


def row_rel(got, want):
    """Reference metric (harness.py:189-206); NaN/Inf count as infinite error
    (the reference guards finiteness separately, harness.py:289-290)."""
    got = np.asarray(got, dtype=np.float64)
    if not np.isfinite(got).all():
        return float("inf"), float("inf")
    return oh.output_errors([got], [want])
