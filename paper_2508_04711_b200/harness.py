"""Synthetic jagged batches and the error metric (mirror of
``jaggedcp/harness.py``: harness.py:52-206).

``gen_synthetic_batch`` draws from the same numpy RNG stream as the
reference (``default_rng([seed, rank])``: lengths, q, k, v, starts, gaps in
that order), so a config produces the reference's exact inputs; values are
then rounded to bf16 on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .attention import BiasConfig, BiasParams
from .jagged import new_int_series, new_jagged

PROTOCOLS = ("allgather_split", "alltoall")
LENGTH_DISTS = ("uniform", "lognormal")
MAX_TS_GAP_SECONDS = 1_000_000


@dataclass(frozen=True)
class ExperimentConfig:
    """harness.py:52-95 (+ num_heads)."""

    cp_size: int = 2
    batch_size: int = 2
    length_dist: str = "uniform"
    min_len: int = 1
    max_len: int = 32
    lognorm_mu: float = 3.0
    lognorm_sigma: float = 0.8
    max_length: int = 128
    embed_dim: int = 8
    num_buckets: int = 16
    dtype: str = "bf16"
    protocol: str = "alltoall"
    balance_mode: str = "balanced_minichunk"
    seed: int = 0
    num_heads: int = 1

    def __post_init__(self) -> None:
        if self.cp_size < 1:
            raise ValueError("cp_size must be >= 1")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.length_dist not in LENGTH_DISTS:
            raise ValueError(f"unknown length_dist {self.length_dist!r}")
        if self.length_dist == "uniform" and not (0 <= self.min_len <= self.max_len <= self.max_length):
            raise ValueError("degenerate distribution bounds: need 0 <= min_len <= max_len <= max_length")
        if self.length_dist == "lognormal" and self.lognorm_sigma < 0:
            raise ValueError("degenerate distribution bounds: lognorm_sigma must be >= 0")
        if self.embed_dim < 1 or self.num_buckets < 1 or self.max_length < 1:
            raise ValueError("embed_dim, num_buckets and max_length must be >= 1")
        if self.protocol not in PROTOCOLS:
            raise ValueError(f"protocol must be one of {PROTOCOLS}")
        if self.balance_mode not in ("balanced_minichunk", "naive_contiguous"):
            raise ValueError("unknown balance_mode")


def draw_lengths(cfg: ExperimentConfig, rng: np.random.Generator) -> np.ndarray:
    """harness.py:116-120."""
    if cfg.length_dist == "uniform":
        return rng.integers(cfg.min_len, cfg.max_len + 1, size=cfg.batch_size)
    raw = np.floor(rng.lognormal(cfg.lognorm_mu, cfg.lognorm_sigma, size=cfg.batch_size))
    return np.clip(raw, 1, cfg.max_length).astype(np.int64)


def gen_synthetic_host(cfg: ExperimentConfig, rank: int) -> dict:
    """harness.py:123-145 on the host: dict of numpy arrays (q/k/v f32)."""
    rng = np.random.default_rng([cfg.seed, rank])
    seq_lengths = draw_lengths(cfg, rng)
    offsets = np.concatenate([[0], np.cumsum(seq_lengths)]).astype(np.int64)
    total = int(offsets[-1])
    q = rng.standard_normal((total, cfg.embed_dim), dtype=np.float32)
    k = rng.standard_normal((total, cfg.embed_dim), dtype=np.float32)
    v = rng.standard_normal((total, cfg.embed_dim), dtype=np.float32)
    starts = rng.integers(0, 1_000_000_000, size=cfg.batch_size)
    gaps = rng.integers(1, MAX_TS_GAP_SECONDS + 1, size=total)
    ts = np.zeros(total, dtype=np.int64)
    for b in range(cfg.batch_size):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        ts[lo:hi] = starts[b] + np.cumsum(gaps[lo:hi])
    return {"q": q, "k": k, "v": v, "ts": ts, "offsets": offsets}


def gen_synthetic_batch(cfg: ExperimentConfig, rank: int, device=None):
    """harness.py:123-145 -> cp_engine.QKVBatch on the GPU (bf16 values)."""
    from .cp_engine import QKVBatch
    h = gen_synthetic_host(cfg, rank)
    return QKVBatch(
        q=new_jagged(h["q"], h["offsets"], cfg.max_length, device),
        k=new_jagged(h["k"], h["offsets"], cfg.max_length, device),
        v=new_jagged(h["v"], h["offsets"], cfg.max_length, device),
        ts=new_int_series(h["ts"], h["offsets"], device),
    )


def bias_for_config(cfg: ExperimentConfig):
    """harness.py:148-152 (seed + 0x5EED)."""
    bias_cfg = BiasConfig(num_buckets=cfg.num_buckets)
    return BiasParams.normal_init(bias_cfg, seed=cfg.seed + 0x5EED), bias_cfg


def output_errors(got, want) -> tuple[float, float]:
    """harness.py:189-206: (max abs, max row-normalized error)."""
    max_abs = max_rel = 0.0
    for g, w in zip(got, want):
        g = g.values if hasattr(g, "values") else g
        w = w.values if hasattr(w, "values") else w
        g = g.detach().float().cpu().numpy() if isinstance(g, torch.Tensor) else np.asarray(g, np.float64)
        w = w.detach().float().cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w, np.float64)
        if g.shape[0] == 0:
            continue
        diff = np.abs(g.astype(np.float64) - w.astype(np.float64))
        ref = np.abs(w.astype(np.float64))
        max_abs = max(max_abs, float(diff.max()))
        max_rel = max(max_rel, float((diff.max(axis=1) / np.maximum(1.0, ref.max(axis=1))).max()))
    return max_abs, max_rel
