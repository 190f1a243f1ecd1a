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
        t = torch.from_numpy(np.ascontiguousarray(self.ts_weights, dtype=np.float32))
        if torch.device(device).type == "cuda":  # (pinned: a pageable copy would wait for the stream)
            t = t.pin_memory()
        return t.to(device, non_blocking=True)


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


def _host_i64(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.int64).reshape(-1)


def _dev_rows(x, dtype, device) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device=device, dtype=dtype).contiguous()


def _blockwise_segments(q_seq_ids, q_positions, k_seq_ids, k_positions):
    """Host routing of blockwise_partial onto the kernel's segment form.

    The keys are sorted by (sequence, position).  A query of sequence s gets an
    effective position e in s's sorted key run: e = q_pos - p0 when the run's
    positions are consecutive p0, p0+1, ... (e may exceed the run: every key
    visible), otherwise e = vis - 1 with vis = #keys of s at positions <= q_pos.
    Either way the query sees exactly the run's keys 0..e, i.e. the
    reference's allowed set (attention.py:180-183).  Queries sorted by (s, e)
    with consecutive e share one segment (q_pos0 = e of its first row,
    kv = s's run); queries with e < 0 see nothing and get kv_len 0.  Returns
    (q_perm, k_perm, q_offsets, q_pos0, kv_start, kv_len)."""
    qs, qp, ks, kp = (_host_i64(x) for x in (q_seq_ids, q_positions, k_seq_ids, k_positions))
    k_perm = np.lexsort((kp, ks))
    ks_s, kp_s = ks[k_perm], kp[k_perm]
    seqs, run_start = np.unique(ks_s, return_index=True)
    run_len = np.diff(np.append(run_start, ks_s.size))
    eff = np.full(qs.size, -1, dtype=np.int64)
    rs = np.zeros(qs.size, dtype=np.int64)
    rl = np.zeros(qs.size, dtype=np.int64)
    if seqs.size:
        j = np.searchsorted(seqs, qs)
        jj = np.minimum(j, seqs.size - 1)
        has = (j < seqs.size) & (seqs[jj] == qs)
        consec = {}
        for i in np.nonzero(has)[0]:
            a, n = int(run_start[jj[i]]), int(run_len[jj[i]])
            rs[i], rl[i] = a, n
            if a not in consec:
                consec[a] = bool(np.all(np.diff(kp_s[a:a + n]) == 1))
            if consec[a]:
                eff[i] = qp[i] - kp_s[a]
            else:
                eff[i] = np.searchsorted(kp_s[a:a + n], qp[i], side="right") - 1
    eff = np.maximum(eff, -1)
    q_perm = np.lexsort((eff, qs))
    offs, pos0, kvs, kvl = [0], [], [], []
    prev = None  # (sequence, eff) of the previous query row in q_perm order
    for row, i in enumerate(q_perm):
        if prev is None or qs[i] != prev[0]:
            new = True
        elif eff[i] < 0:
            new = False  # (sorted: a sequence's blind rows come first, one kv_len-0 segment)
        else:
            new = prev[1] < 0 or eff[i] != prev[1] + 1
        if new and row > 0:
            offs.append(row)
        if new:
            pos0.append(max(int(eff[i]), 0))
            kvs.append(int(rs[i]))
            kvl.append(int(rl[i]) if eff[i] >= 0 else 0)
        prev = (qs[i], eff[i])
    if qs.size:
        offs.append(qs.size)
    a64 = lambda x: np.asarray(x, dtype=np.int64)  # noqa: E731
    return q_perm.astype(np.int64), k_perm.astype(np.int64), a64(offs), a64(pos0), a64(kvs), a64(kvl)


def blockwise_partial(q, q_seq_ids, q_positions, ts_q, k, k_seq_ids, k_positions, ts_k, v,
                      params: BiasParams, cfg: BiasConfig) -> torch.Tensor:
    """attention.py:151-184 -- attention contribution of one key/value block to
    one query block: a pair (i, j) contributes iff both rows are in the same
    sequence and k_positions[j] <= q_positions[i].  SiLU partials are additive,
    so the full output is the plain sum of these over any key partition.

    Runs the fused sm_100a forward in its segment form (fp32 output): keys are
    sorted by (sequence, position) on the host plan, rows are moved by the
    gather / scatter kernels.  Returns a float32 CUDA tensor (nq, d)."""
    kn = k.shape[0]
    vn = v.shape[0]
    if kn != vn:
        raise ValueError(f"k has {kn} rows but v has {vn}")
    nq = q.shape[0]
    dv = v.shape[1] if len(v.shape) == 2 else 0
    dev = q.device if isinstance(q, torch.Tensor) and q.is_cuda else torch.device("cuda")
    if nq == 0 or kn == 0:
        return torch.zeros((nq, dv), dtype=torch.float32, device=dev)
    if q.shape[1] != k.shape[1] or dv != q.shape[1]:
        raise ValueError("q, k, v must share embed_dim")
    q_perm, k_perm, offs, pos0, kvs, kvl = _blockwise_segments(q_seq_ids, q_positions, k_seq_ids, k_positions)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    qp, kp = t(q_perm), t(k_perm)
    qd = kernels.gather_rows(_dev_rows(q, torch.bfloat16, dev), qp)
    kd = kernels.gather_rows(_dev_rows(k, torch.bfloat16, dev), kp)
    vd = kernels.gather_rows(_dev_rows(v, torch.bfloat16, dev), kp)
    tq = kernels.gather_rows(_dev_rows(_host_i64(ts_q), torch.int64, dev).view(-1, 1), qp).view(-1)
    tk = kernels.gather_rows(_dev_rows(_host_i64(ts_k), torch.int64, dev).view(-1, 1), kp).view(-1)
    acc = torch.empty((nq, qd.shape[1]), dtype=torch.float32, device=dev)
    kernels.attn_fwd(qd, kd, vd, tq, tk, t(offs), 1, params.device_weights(dev), cfg.num_buckets,
                     q_pos0=t(pos0), kv_start=t(kvs), kv_len=t(kvl), kv_len_total=int(kvl.sum()),
                     out_accum=acc)
    return kernels.scatter_rows(acc, qp, torch.empty_like(acc))


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
                                            seg_host=(q.host_offsets, None, None))
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


# ------------------------------------------------------------ host streaming

def _as_pinned(x, dtype):
    """Host tensor in page-locked memory (a zero-copy view when it already is)."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if t.is_cuda:
        raise ValueError("host streaming takes host (CPU) buffers")
    t = t.to(dtype) if t.dtype != dtype else t
    return t if t.is_pinned() else t.pin_memory()


_STREAMS: dict = {}
_PIN_RING: dict = {}
_PIN_SLOTS = 8


class _PinSlot:
    """Page-locked staging buffers of one in-flight host-streaming call
    (segment offsets, ts_weights, d_ts_weights).  Allocating page-locked memory
    per call stalled the host for tens of ms in the first calls of a process
    (scripts/e2e_pipe_probe.py); a ring of slots reuses them once the call that
    last used the slot has finished."""

    def __init__(self):
        self.event = None
        self.bufs = {}

    def get(self, name, n, dtype):
        b = self.bufs.get(name)
        if b is None or b.numel() < n or b.dtype != dtype:
            b = torch.empty(max(n, 64), dtype=dtype, pin_memory=True)
            self.bufs[name] = b
        return b[:n]


def _pin_slot(dev) -> _PinSlot:
    ring = _PIN_RING.setdefault(dev, {"slots": [_PinSlot() for _ in range(_PIN_SLOTS)], "k": 0})
    slot = ring["slots"][ring["k"] % _PIN_SLOTS]
    ring["k"] += 1
    if slot.event is not None:
        slot.event.synchronize()  # (normally long done: _PIN_SLOTS calls ago)
    return slot


def _stream_cuts(offs: np.ndarray, G: int) -> list:
    """Sequence-boundary cut points of G runs with ~T/G tokens each (unequal
    first / last runs were measured: no gain, the PCIe rates bind)."""
    B, T = offs.size - 1, int(offs[-1])
    cuts = [0]
    for gi in range(1, G):
        b = int(np.searchsorted(offs, gi * T / G))
        cuts.append(min(max(b, cuts[-1] + 1), B - (G - gi)))
    cuts.append(B)
    return cuts


class HostStreamResult:
    """Handle of an enqueued host-streaming call: ``wait()`` blocks until every
    result reached the host and returns (out, dq, dk, dv, d_ts_weights)."""

    def __init__(self, event, results, keep):
        self._event, self._results, self._keep = event, results, keep

    def done(self) -> bool:
        return self._event.query()

    def wait(self):
        self._event.synchronize()
        self._keep = None
        r = self._results
        return r[0], r[1], r[2], r[3], r[4].clone()  # (d_ts_weights: out of the reused staging slot)


def hstu_attention_fwd_bwd_host_async(q, k, v, ts, offsets, upstream, ts_weights, num_heads: int = 1,
                                      num_buckets: int = 16, groups: int = 4, device=None, out=None):
    """Enqueue hstu_attention_fwd_bwd_host without waiting: returns a
    HostStreamResult.  Consecutive calls overlap -- one call's results copy
    back while the next call's inputs copy in (PCIe is full duplex) -- as long
    as calls in flight write different ``out`` buffers (a caller double-
    buffers them, and waits for call i before reusing call i's buffers)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    offs = np.asarray(offsets.cpu() if isinstance(offsets, torch.Tensor) else offsets, dtype=np.int64)
    if offs.ndim != 1 or offs.size < 1 or offs[0] != 0 or np.any(np.diff(offs) < 0):
        raise ValueError("offsets must start at 0 and be monotone")
    T = int(offs[-1])
    qh, kh, vh, gh = (_as_pinned(x, torch.bfloat16) for x in (q, k, v, upstream))
    tsh = _as_pinned(ts, torch.int64)
    for name, x in (("q", qh), ("k", kh), ("v", vh), ("upstream", gh)):
        if x.dim() != 2 or x.shape[0] != T or x.shape != qh.shape:
            raise ValueError(f"{name} must be (T, H*d) with T = offsets[-1] = {T} rows like q")
    if tsh.shape != (T,):
        raise ValueError("ts must have one timestamp per row")
    B = offs.size - 1
    G = max(1, min(int(groups), B))
    cuts = _stream_cuts(offs, G)
    if out is not None:
        outs = list(out)
        if len(outs) != 4 or any(o.shape != qh.shape or o.dtype != torch.bfloat16 or not o.is_pinned() for o in outs):
            raise ValueError("out must be four pinned bf16 host tensors shaped like q")
    else:
        outs = [torch.empty(qh.shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
    if dev not in _STREAMS:
        _STREAMS[dev] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    s_in, s_out = _STREAMS[dev]
    main = torch.cuda.current_stream(dev)
    runs = []
    slot = _pin_slot(dev)
    subs = [offs[cuts[gi]:cuts[gi + 1] + 1] - offs[cuts[gi]] for gi in range(G)]
    pos = [0]
    for x in subs:  # each run's offsets at a 64-byte aligned position
        pos.append(pos[-1] + (x.size + 7) // 8 * 8)
    offs_pin = slot.get("offs", pos[-1], torch.int64)
    for x, p0 in zip(subs, pos):
        offs_pin.numpy()[p0:p0 + x.size] = x
    # (no wait on the caller's stream: the copies read host memory into fresh
    # buffers, so the next call's inputs can copy in while this one still runs)
    with torch.cuda.stream(s_in):
        offs_dev = offs_pin.to(dev, non_blocking=True)
        offs_dev.record_stream(main)
        # every run's inputs are enqueued first, so the host's launch overhead of the
        # runs below overlaps the copies instead of delaying them; the device inputs
        # are allocated once and filled run by run (slice copies into one buffer run
        # at the full PCIe rate; per-slice .to() allocations measured ~25 % slower)
        dev_in = [torch.empty(x.shape, dtype=x.dtype, device=dev) for x in (qh, kh, vh, gh)]
        for x in dev_in:
            x.record_stream(main)
        for gi in range(G):
            b0, b1 = cuts[gi], cuts[gi + 1]
            r0, r1 = int(offs[b0]), int(offs[b1])
            if r1 == r0:
                continue
            sub = subs[gi]
            ins = []
            for dst, src in zip(dev_in, (qh, kh, vh, gh)):
                dst[r0:r1].copy_(src[r0:r1], non_blocking=True)
                ins.append(dst[r0:r1])
            ins.append(tsh[r0:r1].to(dev, non_blocking=True))  # (its own buffer: 16-byte aligned)
            ins.append(offs_dev[pos[gi]:pos[gi] + sub.size])
            ev = torch.cuda.Event()
            ev.record(s_in)
            runs.append((b0, b1, r0, r1, sub, ins, ev))
    # (after the copies are queued: nothing on the host delays the first one)
    w_np = np.asarray(ts_weights, dtype=np.float32).reshape(-1)
    w_pin = slot.get("w", w_np.size, torch.float32)
    w_pin.numpy()[:] = w_np
    w = w_pin.to(dev, non_blocking=True)
    d_w = torch.zeros(num_buckets, dtype=torch.float64, device=dev)
    keep = []
    for b0, b1, r0, r1, sub, ins, ev in runs:
        main.wait_event(ev)
        for x in ins:
            x.record_stream(main)
        dq_, dk_, dv_, dg_, dts, doffs = ins
        band = kernels.new_band_table(r1 - r0, b1 - b0, dev)
        o = kernels.attn_fwd(dq_, dk_, dv_, dts, dts, doffs, num_heads, w, num_buckets, band_table=band)
        gq, gk, gv, gw, _ = kernels.attn_bwd(dq_, dk_, dv_, dts, dts, doffs, dg_, num_heads, w, num_buckets,
                                             band_table=band, seg_host=(sub, None, None))
        d_w += gw
        s_out.wait_stream(main)
        with torch.cuda.stream(s_out):
            for dst, src in zip(outs, (o, gq, gk, gv)):
                src.record_stream(s_out)
                dst[r0:r1].copy_(src, non_blocking=True)
        keep.append((o, gq, gk, gv))
    dwh = slot.get("dw", num_buckets, torch.float64)
    s_out.wait_stream(main)
    with torch.cuda.stream(s_out):
        d_w.record_stream(s_out)
        dwh.copy_(d_w, non_blocking=True)
        done = torch.cuda.Event()
        done.record(s_out)
    slot.event = done
    return HostStreamResult(done, (outs[0], outs[1], outs[2], outs[3], dwh), keep)


def hstu_attention_fwd_bwd_host(q, k, v, ts, offsets, upstream, ts_weights, num_heads: int = 1,
                                num_buckets: int = 16, groups: int = 4, device=None, out=None):
    """Forward + backward of attention.py:125-148 / 187-234 for inputs that live in
    HOST memory (the reference's numpy calling convention), returning host
    results: (out, dq, dk, dv) as bf16 host tensors shaped like q and
    d_ts_weights (float64, host).

    The batch is cut into ``groups`` runs of whole sequences with about equal
    token counts (sequences never interact, so each run is an independent
    problem); every run's host->device copy is enqueued first on a copy
    stream, each run's kernels start when its inputs land, and its results go
    back on a second copy stream while later runs still copy in, so the two
    PCIe directions overlap each other and the kernels (C2 on one B200: 2.46
    ms vs 2.82 ms for copy-in / compute / copy-out in sequence; PCIe 5 x16,
    ~42 GB/s per direction while both run, 55 alone).  q, k, v, upstream: (T, H*d) host arrays / tensors (bf16, or anything
    castable; pinned tensors are used in place); ts: (T,) int64; offsets:
    (B+1,) int64 host.  ``out`` = four pinned bf16 host tensors shaped like q to
    write (out, dq, dk, dv) into (reused across calls; otherwise allocated)."""
    return hstu_attention_fwd_bwd_host_async(q, k, v, ts, offsets, upstream, ts_weights, num_heads, num_buckets,
                                             groups, device, out).wait()
