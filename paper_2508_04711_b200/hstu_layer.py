"""HSTU layer and stack around the fused attention.

The reference stops at the attention op (SPEC.md:227 lists the layer stack as
a non-goal); configs C4 (8 layers, CP = 8) and C5 need the layer, so it is
built here on the same kernels.  One layer (the HSTU block of arXiv
2402.17152, which arXiv 2508.04711 shards):

    xn   = LN(x) * g_in + b_in                               jh_norm_gate (no gate)
    uvqk = SiLU(xn W1 + b1);  u, v, q, k = split(uvqk)       cuBLAS GEMM + jh_silu
    a    = tril . SiLU((q k^T + bias(ts)) / sqrt(d)) v       fused attention kernels
    y    = (LN(a) * g_out + b_out) * u                       jh_norm_gate (gated)
    out  = x + y W2 + b2                                     cuBLAS GEMM

u, v, q, k are column views of one uvqk buffer (row stride 4 H d): the
attention kernels read them in place through TMA, no split copies.

Under jagged CP (``HSTUStack(cp=CPAttention(...))``) the activations are
redistributed ONCE at the stack input into the resident (plan-order) layout,
every row-wise op and GEMM runs on the resident rows, each layer's attention
exchanges K/V with the CP group (cp_layer.CPAttention.attend), and the output
is restored once at the end -- activations stay sequence-sharded across
layers.  Gradients: ts_weights are summed over the CP group inside the
attention backward; ``cp_grad_sync`` sums every other parameter's gradient
over the CP group (each rank saw different tokens of the same batch), after
which a DDP wrapper over the DP group averages over replicas.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import kernels
from .attention import BiasConfig, BiasParams, hstu_attention


class _SiluFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        ctx.save_for_backward(x)
        return kernels.silu(x)

    @staticmethod
    def backward(ctx, g):
        (x,) = ctx.saved_tensors
        return kernels.silu_bwd(x, g.to(torch.bfloat16).contiguous())


class _NormGateFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, u, gamma, beta, eps):
        y, mean, rstd = kernels.norm_gate_fwd(x, u, gamma, beta, eps)
        ctx.save_for_backward(x, u, gamma, beta, mean, rstd)
        return y

    @staticmethod
    def backward(ctx, g):
        x, u, gamma, beta, mean, rstd = ctx.saved_tensors
        dx, du, dg, db = kernels.norm_gate_bwd(g.to(torch.bfloat16), x, u, gamma, beta, mean, rstd)
        return dx, du, dg, db, None


class _LinearSiluFn(torch.autograd.Function):
    """uvqk = SiLU(xn W + b) as one node: the backward computes d(pre-activation)
    and the bias gradient in one pass (jh_silu_bwd_colsum) instead of a SiLU
    node + autograd's addmm backward re-reading the [rows, 4 H d] gradient for
    the bias sum (r2 C4 stack profile: 8 x 56 us of torch reductions)."""

    @staticmethod
    def forward(ctx, xn, w, b):
        wb = w.to(xn.dtype)
        h = torch.addmm(b.to(xn.dtype), xn, wb)
        ctx.save_for_backward(xn, wb, h)
        return kernels.silu(h)

    @staticmethod
    def backward(ctx, dy):
        xn, wb, h = ctx.saved_tensors
        dh, db = kernels.silu_bwd_colsum(h, dy.to(torch.bfloat16).contiguous())
        dxn = dh @ wb.t() if ctx.needs_input_grad[0] else None
        dw = (xn.t() @ dh).float() if ctx.needs_input_grad[1] else None
        return dxn, dw, db


class _LinearResidualFn(torch.autograd.Function):
    """out = x + y W + b; the bias gradient is a jh_colsum of d out."""

    @staticmethod
    def forward(ctx, y, w, b, x):
        wb = w.to(y.dtype)
        ctx.save_for_backward(y, wb)
        return x + torch.addmm(b.to(y.dtype), y, wb)

    @staticmethod
    def backward(ctx, dout):
        y, wb = ctx.saved_tensors
        dout = dout.to(torch.bfloat16).contiguous()
        dy = dout @ wb.t() if ctx.needs_input_grad[0] else None
        dw = (y.t() @ dout).float() if ctx.needs_input_grad[1] else None
        db = kernels.colsum(dout) if ctx.needs_input_grad[2] else None
        return dy, dw, db, dout


def silu(x):
    return _SiluFn.apply(x)


def norm_gate(x, u, gamma, beta, eps: float = 1e-6):
    """(LN(x) * gamma + beta) * u, u optional (plain LayerNorm)."""
    return _NormGateFn.apply(x, u, gamma, beta, eps)


class _AttnGateFn(torch.autograd.Function):
    """uvqk -> y = (LN(attention(q, k, v)) * g + b) * u as ONE autograd node: its
    backward writes du, dq, dk, dv straight into the column slices of a single
    d(uvqk) buffer (the kernels take any row stride), instead of four tensors
    that autograd's split-backward concatenates (r2 C4 stack profile: 55 us of
    copy per layer)."""

    @staticmethod
    def forward(ctx, uvqk, ts, offsets, w, gamma, beta, num_heads, num_buckets, max_len, eps):
        n = uvqk.shape[1] // 4
        u, v, q, k = uvqk.split(n, dim=1)
        band = kernels.new_band_table(q.shape[0], offsets.numel() - 1, q.device)
        a = kernels.attn_fwd(q, k, v, ts, ts, offsets, num_heads, w, num_buckets, band_table=band)
        y, mean, rstd = kernels.norm_gate_fwd(a, u, gamma, beta, eps)
        ctx.save_for_backward(uvqk, ts, offsets, w, gamma, beta, a, mean, rstd)
        ctx.band, ctx.cfg = band, (num_heads, num_buckets, max_len)
        return y

    @staticmethod
    def backward(ctx, dy):
        uvqk, ts, offsets, w, gamma, beta, a, mean, rstd = ctx.saved_tensors
        H, nb, max_len = ctx.cfg
        n = uvqk.shape[1] // 4
        u, v, q, k = uvqk.split(n, dim=1)
        g = torch.empty_like(uvqk)
        gu, gv, gq, gk = g.split(n, dim=1)
        da, _, dgam, dbet = kernels.norm_gate_bwd(dy.to(torch.bfloat16).contiguous(), a, u, gamma, beta, mean, rstd,
                                                  du_out=gu)
        _, _, _, dw, _ = kernels.attn_bwd(q, k, v, ts, ts, offsets, da, H, w, nb, max_kv_len=max_len,
                                          band_table=ctx.band, out=(gq, gk, gv))
        return g, None, None, dw.to(w.dtype), dgam, dbet, None, None, None, None


class KernelOps:
    """The layer's row-wise ops on the sm_100a kernels (the product path; tests
    inject a CPU double the same way cp_layer takes a compute backend)."""

    silu = staticmethod(silu)
    norm_gate = staticmethod(norm_gate)

    @staticmethod
    def linear_silu(xn, w, b):
        return _LinearSiluFn.apply(xn, w, b)

    @staticmethod
    def linear_residual(y, w, b, x):
        return _LinearResidualFn.apply(y, w, b, x)

    @staticmethod
    def attention(q, k, v, ts, offsets, w, H, nb, max_len):
        return hstu_attention(q, k, v, ts, offsets, w, H, nb, max_len=max_len)

    @staticmethod
    def attention_gate(uvqk, ts, offsets, w, gamma, beta, H, nb, max_len, eps):
        return _AttnGateFn.apply(uvqk, ts, offsets, w, gamma, beta, H, nb, max_len, eps)


class HSTULayer(torch.nn.Module):
    """One HSTU block (see module docstring).  Parameters are fp32; the GEMMs
    and activations run in bf16 (fp32 accumulation)."""

    def __init__(self, embed_dim: int, num_heads: int, head_dim: int, num_buckets: int = 16, eps: float = 1e-6,
                 seed: int = 0, ops=None):
        super().__init__()
        self.ops = ops if ops is not None else KernelOps
        if embed_dim % 8 or head_dim % 8:
            raise ValueError("embed_dim and head_dim must be multiples of 8")
        self.embed_dim, self.num_heads, self.head_dim = embed_dim, num_heads, head_dim
        self.num_buckets, self.eps = num_buckets, eps
        n = num_heads * head_dim
        gen = torch.Generator().manual_seed(seed)
        self.in_gamma = torch.nn.Parameter(torch.ones(embed_dim))
        self.in_beta = torch.nn.Parameter(torch.zeros(embed_dim))
        self.w_uvqk = torch.nn.Parameter(torch.randn(embed_dim, 4 * n, generator=gen) / math.sqrt(embed_dim))
        self.b_uvqk = torch.nn.Parameter(torch.zeros(4 * n))
        w = BiasParams.normal_init(BiasConfig(num_buckets), seed).ts_weights
        self.ts_weights = torch.nn.Parameter(torch.from_numpy(np.asarray(w, dtype=np.float32)))
        self.out_gamma = torch.nn.Parameter(torch.ones(n))
        self.out_beta = torch.nn.Parameter(torch.zeros(n))
        self.w_o = torch.nn.Parameter(torch.randn(n, embed_dim, generator=gen) / math.sqrt(n))
        self.b_o = torch.nn.Parameter(torch.zeros(embed_dim))

    def forward(self, x, ts, offsets=None, max_len=None, cp=None):
        """x: (rows, embed_dim) bf16 (local rows, or resident rows under CP);
        ts: (rows,) int64.  Single device: ``offsets`` (B+1,) int64 on the
        device and ``max_len`` (host bound of the lengths).  CP: ``cp`` =
        (CPAttention, plan) from HSTUStack."""
        n = self.num_heads * self.head_dim
        dt, ops = x.dtype, self.ops
        xn = ops.norm_gate(x, None, self.in_gamma, self.in_beta, self.eps)
        if hasattr(ops, "linear_silu"):
            uvqk = ops.linear_silu(xn, self.w_uvqk, self.b_uvqk)
            out_proj = lambda y: ops.linear_residual(y, self.w_o, self.b_o, x)  # noqa: E731
        else:
            uvqk = ops.silu(torch.addmm(self.b_uvqk.to(dt), xn, self.w_uvqk.to(dt)))
            out_proj = lambda y: x + torch.addmm(self.b_o.to(dt), y, self.w_o.to(dt))  # noqa: E731
        if cp is None and hasattr(ops, "attention_gate") and max_len is not None and self.head_dim in (64, 128):
            y = ops.attention_gate(uvqk, ts, offsets, self.ts_weights, self.out_gamma, self.out_beta,
                                   self.num_heads, self.num_buckets, max_len, self.eps)
            return out_proj(y)
        u, v, q, k = uvqk.split(n, dim=1)
        if cp is None:
            a = ops.attention(q, k, v, ts, offsets, self.ts_weights, self.num_heads, self.num_buckets, max_len)
        else:
            from .cp_layer import cp_resident_attention
            layer, plan = cp
            a = cp_resident_attention(layer, plan, q, k, v, ts, self.ts_weights)
        y = ops.norm_gate(a, u, self.out_gamma, self.out_beta, self.eps)
        return out_proj(y)


class HSTUStack(torch.nn.Module):
    """``num_layers`` HSTU blocks; optionally sharded by jagged CP (``cp`` =
    a cp_layer.CPAttention over the CP process group)."""

    def __init__(self, num_layers: int, embed_dim: int, num_heads: int, head_dim: int, num_buckets: int = 16,
                 seed: int = 0, cp=None, ops=None):
        super().__init__()
        self.layers = torch.nn.ModuleList(
            HSTULayer(embed_dim, num_heads, head_dim, num_buckets, seed=seed + 1000 * i, ops=ops)
            for i in range(num_layers))
        self.cp = cp
        if cp is not None and (cp.H != num_heads or cp.nb != num_buckets):
            raise ValueError("CPAttention heads / buckets differ from the stack's")

    def forward(self, x, ts, offsets=None, max_len=None, local_lengths=None):
        """Single device: x (T, embed_dim) bf16, ts (T,), offsets (B+1,) device,
        max_len.  CP: x / ts are this rank's LOCAL rows and ``local_lengths``
        its sequence lengths (host); the output is in the same local layout."""
        if self.cp is None:
            for layer in self.layers:
                x = layer(x, ts, offsets, max_len)
            return x
        from .cp_layer import cp_shard, cp_unshard
        if local_lengths is None:
            raise ValueError("local_lengths is required under CP")
        plan = self.cp.plan_for(np.asarray(local_lengths), x.device)
        n_local = x.shape[0]
        x_r = cp_shard(self.cp, plan, x, n_local)
        ts_r = self.cp.redistribute(ts.view(-1, 1), *plan).view(-1)
        for layer in self.layers:
            x_r = layer(x_r, ts_r, cp=(self.cp, plan))
        return cp_unshard(self.cp, plan, x_r, n_local)

    def cp_grad_sync(self):
        """Sum every non-ts_weights gradient over the CP group (ts_weights are
        already summed by the attention backward).  Call after backward and
        before the DP all-reduce / optimizer step."""
        if self.cp is None:
            return
        for name, p in self.named_parameters():
            if p.grad is not None and not name.endswith("ts_weights"):
                self.cp.comm.all_reduce(p.grad)
