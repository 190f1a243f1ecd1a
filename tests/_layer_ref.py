"""Torch reference of the HSTU layer's pieces (TEST INFRASTRUCTURE).

``TorchOps`` is the CPU double of hstu_layer.KernelOps: LayerNorm / SiLU from
torch.nn.functional and a dense per-sequence HSTU attention whose bias indices
come from the oracle's integer bucketize (attention.py:78-94 restated in
oracle/attention.py), so autograd gives the layer's exact gradients in fp32 /
fp64.  Used by the CPU CP-stack test (as the injected ops) and by the GPU
layer tests (as the reference the kernels are checked against)."""

import math

import numpy as np
import torch
import torch.nn.functional as F

import oracle


def dense_attention(q, k, v, ts, offsets_host, w, H, nb):
    """tril(SiLU((q k^T + w[bucket]) / sqrt(d))) v per sequence and head."""
    T, n = q.shape
    d = n // H
    ts_h = ts.detach().cpu().numpy()
    outs = []
    for b in range(len(offsets_host) - 1):
        lo, hi = int(offsets_host[b]), int(offsets_host[b + 1])
        L = hi - lo
        if L == 0:
            continue
        bk = torch.from_numpy(oracle.bucketize_array(ts_h[lo:hi, None] - ts_h[None, lo:hi], nb)).to(q.device)
        bias = w.to(q.dtype)[bk]
        mask = torch.tril(torch.ones(L, L, dtype=torch.bool, device=q.device))
        heads = []
        for h in range(H):
            c = slice(h * d, (h + 1) * d)
            s = (q[lo:hi, c] @ k[lo:hi, c].T + bias) / math.sqrt(d)
            heads.append(torch.where(mask, F.silu(s), torch.zeros_like(s)) @ v[lo:hi, c])
        outs.append(torch.cat(heads, dim=1))
    return torch.cat(outs, dim=0) if outs else q.new_zeros((0, n))


class TorchOps:
    """hstu_layer.KernelOps double on plain torch (any device / dtype)."""

    offsets_host = None  # set by the caller for the single-device attention

    @staticmethod
    def silu(x):
        return F.silu(x)

    @staticmethod
    def norm_gate(x, u, gamma, beta, eps=1e-6):
        y = F.layer_norm(x, (x.shape[1],), gamma.to(x.dtype), beta.to(x.dtype), eps)
        return y if u is None else y * u

    @classmethod
    def attention(cls, q, k, v, ts, offsets, w, H, nb, max_len):
        offs = cls.offsets_host if cls.offsets_host is not None else offsets.detach().cpu().numpy()
        return dense_attention(q, k, v, ts, offs, w, H, nb)


def copy_params(dst, src):
    """Load src's parameters into dst (same architecture)."""
    with torch.no_grad():
        for (n1, p1), (n2, p2) in zip(dst.named_parameters(), src.named_parameters()):
            assert n1 == n2
            p1.copy_(p2.to(p1.dtype))
