"""SiLU-gated causal jagged attention with a learnable time-delta bias, on B200.

Mirror of ``jaggedcp/attention.py`` (/root/reference/pkg/src/jaggedcp/
attention.py): same names, argument meaning and errors, backed by the fused
sm_100a kernels of libjh_hstu.so.

* ``hstu_attention_reference``  (attention.py:125) -> ``jh_attn_fwd``
* ``hstu_attention_backward``   (attention.py:187) -> ``jh_attn_bwd``
* ``bucketize`` / ``compute_bias`` (attention.py:78-94) -> ``jh_bucketize`` /
  ``jh_compute_bias`` (bit-exact integer bucketization)

Extensions (default off, reference semantics unchanged when unused):
``num_heads`` (per-head attention over column blocks, bias shared by heads,
scale sqrt(head_dim)) and ``pos_weights`` (positional bias
``pos_weights[min(i-j, P-1)]``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels
from .jagged import JaggedIntSeries, JaggedTensor


@dataclass(frozen=True)
class BiasConfig:
    """attention.py:21-34."""

    num_buckets: int = 16

    def __post_init__(self) -> None:
        if self.num_buckets < 1:
            raise ValueError("num_buckets must be >= 1")


@dataclass(frozen=True)
class BiasParams:
    """attention.py:37-53: per-bucket weights (host f64, device fp32 copy)."""

    ts_weights: np.ndarray

    @staticmethod
    def normal_init(cfg: BiasConfig, seed: int, mean: float = 0.0, stddev: float = 0.02) -> "BiasParams":
        rng = np.random.default_rng(seed)
        return BiasParams(rng.normal(mean, stddev, size=cfg.num_buckets).astype(np.float64))

    def __post_init__(self) -> None:
        w = self.ts_weights
        w = w.detach().cpu().numpy() if isinstance(w, torch.Tensor) else np.array(w, dtype=np.float64)
        w = np.asarray(w, dtype=np.float64)
        if w.ndim != 1 or w.size < 1:
            raise ValueError("ts_weights must be a non-empty 1-D vector")
        w.setflags(write=False)
        object.__setattr__(self, "ts_weights", w)

    def device_weights(self, device) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(self.ts_weights, dtype=np.float32)).to(device, non_blocking=True)


def silu(x):
    """attention.py:56-66 on a CUDA tensor (x * sigmoid(x))."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ValueError("silu expects a CUDA tensor (there is no CPU path)")
    return torch.nn.functional.silu(x)


def bucketize(delta: int, cfg: BiasConfig) -> int:
    """attention.py:78-80 (one delta, evaluated by the GPU bucket kernel)."""
    d = torch.tensor([int(delta)], dtype=torch.int64, device="cuda")
    return int(kernels.bucketize(d, cfg.num_buckets)[0])


def bucketize_array(deltas, cfg: BiasConfig) -> torch.Tensor:
    """attention.py:83-86 on the GPU (int32 bucket indices)."""
    d = deltas if isinstance(deltas, torch.Tensor) else torch.from_numpy(np.asarray(deltas, dtype=np.int64))
    return kernels.bucketize(d.to("cuda", torch.int64), cfg.num_buckets)


def compute_bias(ts_q, ts_k, params: BiasParams, cfg: BiasConfig) -> torch.Tensor:
    """attention.py:89-94: |q| x |k| fp32 matrix of selected bias weights."""
    tq = ts_q if isinstance(ts_q, torch.Tensor) else torch.from_numpy(np.asarray(ts_q, dtype=np.int64))
    tk = ts_k if isinstance(ts_k, torch.Tensor) else torch.from_numpy(np.asarray(ts_k, dtype=np.int64))
    dev = tq.device if tq.is_cuda else torch.device("cuda")
    return kernels.compute_bias(tq.to(dev, torch.int64), tk.to(dev, torch.int64), params.device_weights(dev),
                                cfg.num_buckets)


@dataclass(frozen=True)
class AttentionInputs:
    """attention.py:97-114 (+ num_heads / pos_weights extensions)."""

    q: JaggedTensor
    k: JaggedTensor
    v: JaggedTensor
    ts: JaggedIntSeries
    params: BiasParams
    cfg: BiasConfig
    num_heads: int = 1
    pos_weights: np.ndarray | None = field(default=None)

    def __post_init__(self) -> None:
        offs = self.q.host_offsets
        for name, other in (("k", self.k), ("v", self.v), ("ts", self.ts)):
            if not np.array_equal(offs, other.host_offsets):
                raise ValueError(f"offsets of q and {name} differ")
        if self.q.embed_dim < 1:
            raise ValueError("embed_dim must be >= 1")
        if self.k.embed_dim != self.q.embed_dim or self.v.embed_dim != self.q.embed_dim:
            raise ValueError("q, k, v must share embed_dim")
        if self.num_heads < 1 or self.q.embed_dim % self.num_heads:
            raise ValueError("embed_dim must be divisible by num_heads")


@dataclass(frozen=True)
class AttentionGradients:
    """attention.py:117-122."""

    dq: JaggedTensor
    dk: JaggedTensor
    dv: JaggedTensor
    d_ts_weights: torch.Tensor  # (num_buckets,) float64, on device
    d_pos_weights: torch.Tensor | None = None


def _pw(inputs: AttentionInputs, device):
    if inputs.pos_weights is None:
        return None
    return torch.as_tensor(np.asarray(inputs.pos_weights, dtype=np.float32)).to(device)


def hstu_attention_reference(inputs: AttentionInputs) -> JaggedTensor:
    """attention.py:125-148 -- fused sm_100a forward (jh_attn_fwd)."""
    q, k, v, ts = inputs.q, inputs.k, inputs.v, inputs.ts
    dev = q.values.device
    out = kernels.attn_fwd(q.values, k.values, v.values, ts.values, ts.values, q.offsets, inputs.num_heads,
                           inputs.params.device_weights(dev), inputs.cfg.num_buckets, _pw(inputs, dev))
    return JaggedTensor(out, q.offsets, v.max_length, q.host_offsets)


def hstu_attention_backward(inputs: AttentionInputs, upstream: JaggedTensor) -> AttentionGradients:
    """attention.py:187-234 -- fused sm_100a backward (jh_attn_bwd)."""
    q, k, v, ts = inputs.q, inputs.k, inputs.v, inputs.ts
    if not np.array_equal(upstream.host_offsets, q.host_offsets):
        raise ValueError("upstream offsets differ from input offsets")
    if tuple(upstream.values.shape) != tuple(v.values.shape):
        raise ValueError("upstream shape differs from output shape")
    dev = q.values.device
    g = upstream.values
    if g.dtype != torch.bfloat16:
        g = g.to(torch.bfloat16)
    dq, dk, dv, dw, dpos = kernels.attn_bwd(q.values, k.values, v.values, ts.values, ts.values, q.offsets,
                                            g.contiguous(), inputs.num_heads, inputs.params.device_weights(dev),
                                            inputs.cfg.num_buckets, _pw(inputs, dev),
                                            max_kv_len=int(np.diff(q.host_offsets).max(initial=0)))
    mk = lambda t, like: JaggedTensor(t, like.offsets, like.max_length, like.host_offsets)  # noqa: E731
    return AttentionGradients(mk(dq, q), mk(dk, k), mk(dv, v), dw, dpos)


# ----------------------------------------------------------------- autograd

class _HSTUAttentionFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, ts_weights, ts, offsets, num_heads, num_buckets, pos_weights, max_len):
        band = kernels.new_band_table(q.shape[0], offsets.numel() - 1, q.device) if pos_weights is None else None
        out = kernels.attn_fwd(q, k, v, ts, ts, offsets, num_heads, ts_weights, num_buckets, pos_weights,
                               band_table=band)
        ctx.save_for_backward(q, k, v, ts_weights, ts, offsets, pos_weights)
        ctx.num_heads, ctx.num_buckets, ctx.band, ctx.max_len = num_heads, num_buckets, band, max_len
        return out

    @staticmethod
    def backward(ctx, g):
        q, k, v, w, ts, offsets, pw = ctx.saved_tensors
        dq, dk, dv, dw, dpos = kernels.attn_bwd(q, k, v, ts, ts, offsets, g.to(torch.bfloat16).contiguous(),
                                                ctx.num_heads, w, ctx.num_buckets, pw, band_table=ctx.band,
                                                max_kv_len=ctx.max_len)
        return (dq, dk, dv, dw.to(w.dtype), None, None, None, None,
                None if dpos is None else dpos.to(pw.dtype), None)


def hstu_attention(q, k, v, ts, offsets, ts_weights, num_heads=1, num_buckets=None, pos_weights=None,
                   max_len=None):
    """Differentiable jagged HSTU attention on device tensors.

    q, k, v: (T, H*d) bf16; ts: (T,) int64; offsets: (B+1,) int64 (device);
    ts_weights: (nb,) parameter.  Gradients flow to q, k, v, ts_weights (and
    pos_weights).  ``max_len`` (an upper bound of the sequence lengths, e.g.
    the JaggedTensor's max_length) keeps the step free of host synchronisation;
    without it the backward reads the longest length back from the device once."""
    nb = ts_weights.numel() if num_buckets is None else int(num_buckets)
    return _HSTUAttentionFn.apply(q, k, v, ts_weights, ts, offsets, int(num_heads), nb, pos_weights,
                                  None if max_len is None else int(max_len))


class JaggedHSTUAttention(torch.nn.Module):
    """The attention "layer": learnable ts_weights (+ optional pos_weights)
    around the fused kernels.  With ``cp_group`` set, the sequence dimension is
    sharded by the jagged CP engine (cp_engine.CPAttention)."""

    def __init__(self, num_heads: int, num_buckets: int = 16, num_pos: int = 0, seed: int | None = None):
        super().__init__()
        w = BiasParams.normal_init(BiasConfig(num_buckets), 0 if seed is None else seed).ts_weights
        self.ts_weights = torch.nn.Parameter(torch.from_numpy(w.astype(np.float32)))
        self.pos_weights = torch.nn.Parameter(torch.zeros(num_pos)) if num_pos else None
        self.num_heads = num_heads
        self.num_buckets = num_buckets

    def forward(self, q, k, v, ts, offsets, max_len=None):
        return hstu_attention(q, k, v, ts, offsets, self.ts_weights, self.num_heads, self.num_buckets,
                              self.pos_weights, max_len)
