"""Torch-facing launchers for the C ABI (libjh_hstu.so).

Every function here takes CUDA tensors, validates dtype/device/shape, allocates
outputs and scratch with the torch caching allocator, and launches on the
current torch stream through ``_lib``.  No CPU path exists: a non-CUDA tensor
or a missing library raises.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import JhAttnArgs, check

_LAUNCHES = {"count": 0}


def launch_count() -> int:
    """Number of jh_* GPU entry points invoked (bench gpu_launches accounting)."""
    return _LAUNCHES["count"]


def _bump(n: int = 1) -> None:
    _LAUNCHES["count"] += n


def _stream(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _require_cuda(name: str, t: torch.Tensor, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def _rowmajor(name: str, t: torch.Tensor):
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be 2-D with unit column stride")


# ----------------------------------------------------------------------- bias

_TABLE_CACHE: dict[int, tuple[np.ndarray, np.ndarray, int]] = {}


def bias_table(num_buckets: int):
    """(thr[64], base[64], cap): the bit-exact octave table (host)."""
    if num_buckets not in _TABLE_CACHE:
        thr = (ctypes.c_int64 * 64)()
        base = (ctypes.c_int32 * 64)()
        cap = ctypes.c_int64()
        check(_lib.lib().jh_bias_table_build(int(num_buckets), thr, base, ctypes.byref(cap)), "bias_table")
        _TABLE_CACHE[num_buckets] = (np.array(thr[:], dtype=np.int64), np.array(base[:], dtype=np.int32), cap.value)
    return _TABLE_CACHE[num_buckets]


def bucketize(deltas: torch.Tensor, num_buckets: int) -> torch.Tensor:
    _require_cuda("deltas", deltas, torch.int64)
    d = deltas.contiguous()
    out = torch.empty(d.shape, dtype=torch.int32, device=d.device)
    check(_lib.lib().jh_bucketize(_ptr(d), d.numel(), int(num_buckets), _ptr(out), _stream(d)), "bucketize")
    _bump()
    return out


def compute_bias(ts_q: torch.Tensor, ts_k: torch.Tensor, ts_weights: torch.Tensor, num_buckets: int) -> torch.Tensor:
    _require_cuda("ts_q", ts_q, torch.int64)
    _require_cuda("ts_k", ts_k, torch.int64)
    w = ts_weights.to(device=ts_q.device, dtype=torch.float32).contiguous()
    _check_weights(w, num_buckets)
    tq, tk = ts_q.contiguous(), ts_k.contiguous()
    out = torch.empty((tq.numel(), tk.numel()), dtype=torch.float32, device=tq.device)
    check(_lib.lib().jh_compute_bias(_ptr(tq), tq.numel(), _ptr(tk), tk.numel(), _ptr(w), int(num_buckets),
                                     _ptr(out), _stream(tq)), "compute_bias")
    _bump()
    return out


def dbias_scatter(ts_q, ts_k, dbias: torch.Tensor, num_buckets: int, d_w: torch.Tensor | None = None):
    _require_cuda("dbias", dbias, torch.float32)
    tq, tk, db = ts_q.contiguous(), ts_k.contiguous(), dbias.contiguous()
    if d_w is None:
        d_w = torch.zeros(num_buckets, dtype=torch.float64, device=db.device)
    check(_lib.lib().jh_dbias_scatter(_ptr(tq), tq.numel(), _ptr(tk), tk.numel(), _ptr(db), int(num_buckets),
                                      _ptr(d_w), _stream(db)), "dbias_scatter")
    _bump()
    return d_w


# ------------------------------------------------------------------ row moves

def gather_rows(src: torch.Tensor, perm: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = src[perm[i]] (jagged.py:244 ``jt.values[perm]``)."""
    _require_cuda("src", src)
    _require_cuda("perm", perm, torch.int64)
    s = src.contiguous()
    rows = perm.numel()
    if out is None:
        out = torch.empty((rows,) + tuple(s.shape[1:]), dtype=s.dtype, device=s.device)
    if rows:
        row_bytes = s.stride(0) * s.element_size()
        check(_lib.lib().jh_gather_rows(_ptr(s), _ptr(out), _ptr(perm), rows, row_bytes, _stream(s)), "gather_rows")
        _bump()
    return out


def scatter_rows(src: torch.Tensor, perm: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[perm[i]] = src[i] (jagged.py:256-257 ``restored[perm] = values``)."""
    _require_cuda("src", src)
    _require_cuda("perm", perm, torch.int64)
    s = src.contiguous()
    rows = perm.numel()
    if out is None:
        out = torch.empty_like(s)
    if rows:
        row_bytes = s.stride(0) * s.element_size()
        check(_lib.lib().jh_scatter_rows(_ptr(s), _ptr(out), _ptr(perm), rows, row_bytes, _stream(s)), "scatter_rows")
        _bump()
    return out


def jagged_to_padded(values: torch.Tensor, offsets: torch.Tensor, max_len: int) -> torch.Tensor:
    _require_cuda("values", values)
    _require_cuda("offsets", offsets, torch.int64)
    v = values.contiguous()
    B = offsets.numel() - 1
    out = torch.empty((B, max_len) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
    row_bytes = (v[0].numel() if v.dim() > 1 else 1) * v.element_size()
    check(_lib.lib().jh_jagged_to_padded(_ptr(v), _ptr(offsets), B, int(max_len), row_bytes, _ptr(out), _stream(v)),
          "jagged_to_padded")
    _bump()
    return out


def padded_to_jagged(padded: torch.Tensor, offsets: torch.Tensor, total: int) -> torch.Tensor:
    _require_cuda("padded", padded)
    _require_cuda("offsets", offsets, torch.int64)
    p = padded.contiguous()
    B, max_len = p.shape[0], p.shape[1]
    out = torch.empty((total,) + tuple(p.shape[2:]), dtype=p.dtype, device=p.device)
    row_bytes = int(np.prod(p.shape[2:])) * p.element_size()
    check(_lib.lib().jh_padded_to_jagged(_ptr(p), _ptr(offsets), B, max_len, row_bytes, _ptr(out), _stream(p)),
          "padded_to_jagged")
    _bump()
    return out


# ------------------------------------------------------------------ attention

def _check_weights(ts_weights, num_buckets, pos_weights=None):
    # the kernels read ts_weights[0 .. num_buckets-1] (attention.py:94 indexes
    # params.ts_weights with buckets < cfg.num_buckets: a shorter vector is an error there too)
    if ts_weights.dim() != 1 or ts_weights.numel() < int(num_buckets):
        raise ValueError(f"ts_weights must be a 1-D vector with at least num_buckets={int(num_buckets)} entries, "
                         f"got shape {tuple(ts_weights.shape)}")
    if pos_weights is not None and (pos_weights.dim() != 1 or pos_weights.numel() < 1):
        raise ValueError("pos_weights must be a non-empty 1-D vector")


def padded_head_dim(d: int) -> int:
    """Head dims the kernels implement: 64 and 128; smaller ones are zero-padded
    (scores keep the 1/sqrt(d) of the true d via score_scale)."""
    if d < 1 or d > 128:
        raise NotImplementedError(f"head_dim {d} unsupported (1 .. 128)")
    return 64 if d <= 64 else 128


def _pad_heads(t, H: int, d: int, dp: int):
    if t is None or d == dp:
        return t
    T = t.shape[0]
    out = t.new_zeros((T, H, dp))
    out[:, :, :d] = t.reshape(T, H, d)
    return out.view(T, H * dp)


def _unpad_heads(t, H: int, d: int, dp: int):
    if t is None or d == dp:
        return t
    return t.view(t.shape[0], H, dp)[:, :, :d].reshape(t.shape[0], H * d)


def _attn_args(q, k, v, ts_q, ts_k, q_offsets, num_heads, ts_weights, num_buckets, pos_weights,
               q_pos0=None, kv_start=None, kv_len=None):
    for name, t in (("q", q), ("k", k), ("v", v)):
        _require_cuda(name, t, torch.bfloat16)
        _rowmajor(name, t)
    for name, t in (("ts_q", ts_q), ("ts_k", ts_k), ("q_offsets", q_offsets), ("q_pos0", q_pos0),
                    ("kv_start", kv_start), ("kv_len", kv_len)):
        if t is None and name not in ("ts_q", "ts_k", "q_offsets"):
            continue
        _require_cuda(name, t, torch.int64)
        if t.dim() != 1 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 1-D tensor")
    if not ts_weights.is_contiguous() or (pos_weights is not None and not pos_weights.is_contiguous()):
        raise ValueError("ts_weights / pos_weights must be contiguous")
    _check_weights(ts_weights, num_buckets, pos_weights)
    D = q.shape[1]
    if D % num_heads:
        raise ValueError(f"embed_dim {D} not divisible by num_heads {num_heads}")
    if k.shape[1] != D or v.shape[1] != D:
        raise ValueError("q, k, v must share embed_dim")
    a = JhAttnArgs()
    a.q, a.k, a.v = q.data_ptr(), k.data_ptr(), v.data_ptr()
    a.ld_q, a.ld_k, a.ld_v = q.stride(0), k.stride(0), v.stride(0)
    a.ts_q, a.ts_k = ts_q.data_ptr(), ts_k.data_ptr()
    a.q_offsets = q_offsets.data_ptr()
    a.q_pos0 = None if q_pos0 is None else q_pos0.data_ptr()
    a.kv_start = None if kv_start is None else kv_start.data_ptr()
    a.kv_len = None if kv_len is None else kv_len.data_ptr()
    a.num_segments = q_offsets.numel() - 1
    a.q_rows = q.shape[0]
    a.kv_rows = k.shape[0]
    a.num_heads = num_heads
    a.head_dim = D // num_heads
    a.ts_weights = ts_weights.data_ptr()
    a.num_buckets = int(num_buckets)
    if pos_weights is not None:
        a.pos_weights = pos_weights.data_ptr()
        a.num_pos = pos_weights.numel()
    return a


def band_table_bytes(q_rows: int, num_segments: int) -> int:
    return int(_lib.lib().jh_attn_band_table_bytes(int(q_rows), int(num_segments)))


def new_band_table(q_rows: int, num_segments: int, device) -> torch.Tensor:
    """Caller-owned band table shared by a forward and a backward call."""
    return torch.empty(band_table_bytes(q_rows, num_segments), dtype=torch.uint8, device=device)


def _band(a, band_table, ready: bool) -> None:
    if band_table is not None:
        if band_table.dtype != torch.uint8 or not band_table.is_cuda:
            raise ValueError("band_table must be a uint8 CUDA tensor (see new_band_table)")
        a.band_table, a.band_table_bytes, a.band_table_ready = band_table.data_ptr(), band_table.numel(), int(ready)


def _workspace(q_rows, kv_total, nseg, H, d, device):
    nbytes = _lib.lib().jh_attn_workspace_bytes(q_rows, kv_total, nseg, H, d)
    return torch.empty(nbytes, dtype=torch.uint8, device=device), nbytes


_TRACE = {"buf": None, "cta": 0}


def set_trace(buf: torch.Tensor | None, cta: int = 0) -> None:
    """Debug timeline: the next attention launches record per-role events of
    CTA ``cta`` into ``buf`` (int64 [5, 4096, 2]: (code<<32 | arg, clock64))."""
    _TRACE["buf"], _TRACE["cta"] = buf, int(cta)


def _prof(a, prof):
    """prof = (start, end) torch.cuda.Event pair recorded around the main kernel."""
    if prof is not None:
        for ev in prof:
            if ev.cuda_event == 0:
                ev.record()  # materialise the event handle
        a.prof_event_start, a.prof_event_end = prof[0].cuda_event, prof[1].cuda_event
    if _TRACE["buf"] is not None:
        a.trace, a.trace_cta = _TRACE["buf"].data_ptr(), _TRACE["cta"]


# The fused kernels take deltas in 32 bits: num_buckets <= 23 (cap e^22 - 1 <
# 2^32).  A larger num_buckets only differs from 23 for pairs whose delta
# reaches bucket 23 (delta >= e^23 - 1 ~ 9.7e9); when the batch's timestamp span
# stays below that, every bucket index is the same under both and the call runs
# with the first 23 weights (d_ts_weights of the higher buckets are 0).
FUSED_NB_MAX = 23


def _effective_buckets(num_buckets: int, ts_q, ts_k) -> int:
    nb = int(num_buckets)
    if nb <= FUSED_NB_MAX or ts_q.numel() == 0 or ts_k.numel() == 0:
        return min(nb, FUSED_NB_MAX) if nb > FUSED_NB_MAX else nb
    span = int((ts_q.max() - ts_k.min()).item())  # >= every pair's delta (one synchronisation)
    if span < bias_table(FUSED_NB_MAX + 1)[2]:  # first delta of bucket 23
        return FUSED_NB_MAX
    raise NotImplementedError(f"fused attention supports num_buckets <= {FUSED_NB_MAX} when a timestamp delta "
                              f"reaches bucket {FUSED_NB_MAX} (num_buckets={nb}, span {span})")


def attn_fwd(q, k, v, ts_q, ts_k, q_offsets, num_heads, ts_weights, num_buckets=16, pos_weights=None,
             q_pos0=None, kv_start=None, kv_len=None, kv_len_total=None, out=None, prof=None, out_accum=None,
             accumulate=False, band_table=None, dbg_buckets=None, band_ready=False):
    """Fused jagged HSTU forward (jh_attn_fwd).  bf16 in/out, fp32 weights.

    ``out_accum`` (fp32, q's shape): write the fp32 result there instead of a
    bf16 ``out`` (``accumulate=True``: add it; rows that see no kv are left
    untouched) -- the additive partials of the CP pipeline (cp_engine.py:441-450).
    ``band_table`` (uint8, ``band_table_bytes``): the near-diagonal bucket table
    is computed into it, for a backward call on the same inputs to reuse
    (``band_ready=True``: it already holds the table, see ``compute_band``).
    Head dims below 64 (or between 64 and 128) are zero-padded; the score scale
    stays 1/sqrt(head_dim).  ``dbg_buckets`` (uint8 [q_rows, max_kv], tests):
    the bucket the kernel applied to each visible pair of head 0."""
    w = ts_weights.to(device=q.device, dtype=torch.float32).contiguous()
    if int(num_buckets) > FUSED_NB_MAX:
        _check_weights(w, num_buckets)
        num_buckets = _effective_buckets(num_buckets, ts_q, ts_k)
        w = w[:num_buckets].contiguous()
    pw = None if pos_weights is None else pos_weights.to(device=q.device, dtype=torch.float32).contiguous()
    H = int(num_heads)
    if q.dim() != 2 or q.shape[1] % H:
        raise ValueError(f"embed_dim {q.shape[-1]} not divisible by num_heads {H}")
    d = q.shape[1] // H
    dp = padded_head_dim(d)
    qq, kk, vv = (_pad_heads(t, H, d, dp) for t in (q, k, v))
    a = _attn_args(qq, kk, vv, ts_q, ts_k, q_offsets, H, w, num_buckets, pw, q_pos0, kv_start, kv_len)
    a.score_scale = 1.0 / float(np.sqrt(d))
    ret = None
    if out_accum is not None:
        if out_accum.dtype != torch.float32 or out_accum.shape != q.shape or out_accum.stride(1) != 1:
            raise ValueError("out_accum must be a float32 tensor shaped like q")
        acc = out_accum
        if dp != d:
            acc = _pad_heads(out_accum, H, d, dp) if accumulate else torch.empty(qq.shape, dtype=torch.float32,
                                                                                  device=q.device)
        a.out_accum, a.ld_o, a.out_accum_mode = acc.data_ptr(), acc.stride(0), 2 if accumulate else 1
        ret = out_accum
    else:
        if out is None:
            out = torch.empty_like(q)
        acc = out if dp == d else torch.empty_like(qq)
        a.out, a.ld_o = acc.data_ptr(), acc.stride(0)
        ret = out
    ws, nbytes = _workspace(q.shape[0], q.shape[0] if kv_len_total is None else kv_len_total, a.num_segments,
                            H, dp, q.device)
    a.workspace, a.workspace_bytes = ws.data_ptr(), nbytes
    _band(a, band_table, ready=band_ready)
    if dbg_buckets is not None:
        if dbg_buckets.dtype != torch.uint8 or dbg_buckets.dim() != 2 or dbg_buckets.shape[0] < q.shape[0] \
                or dbg_buckets.stride(1) != 1:
            raise ValueError("dbg_buckets must be a uint8 [q_rows, max_kv] tensor")
        a.dbg_buckets, a.dbg_ld = dbg_buckets.data_ptr(), dbg_buckets.stride(0)
    _prof(a, prof)
    check(_lib.lib().jh_attn_fwd(ctypes.byref(a), _stream(q)), "hstu_attention forward")
    _bump(2 if (pw is not None or band_ready) else 3)  # (band table) + work-list build + fused forward
    if dp != d:
        ret.copy_(_unpad_heads(acc, H, d, dp))
    return ret


def compute_band(q, ts_q, ts_k, q_offsets, num_heads, num_buckets, band_table, q_pos0=None, kv_start=None,
                 kv_len=None):
    """The near-diagonal bucket table alone (jh_attn_band) into ``band_table``,
    for forward / backward calls with ``band_ready`` / ``band_table``."""
    _require_cuda("band_table", band_table, torch.uint8)
    a = JhAttnArgs()
    for name, t in (("ts_q", ts_q), ("ts_k", ts_k), ("q_offsets", q_offsets)):
        _require_cuda(name, t, torch.int64)
    a.q_offsets, a.ts_q, a.ts_k = q_offsets.data_ptr(), ts_q.data_ptr(), ts_k.data_ptr()
    a.q_pos0 = None if q_pos0 is None else q_pos0.data_ptr()
    a.kv_start = None if kv_start is None else kv_start.data_ptr()
    a.kv_len = None if kv_len is None else kv_len.data_ptr()
    a.num_segments, a.q_rows, a.num_heads = q_offsets.numel() - 1, q.shape[0], int(num_heads)
    a.num_buckets = int(num_buckets)
    a.band_table, a.band_table_bytes = band_table.data_ptr(), band_table.numel()
    check(_lib.lib().jh_attn_band(ctypes.byref(a), _stream(q)), "band table")
    _bump()


_FB_STREAMS: dict = {}


def attn_fwd_bwd(q, k, v, ts, q_offsets, dout, num_heads, ts_weights, num_buckets=16, seg_host=None,
                 band_table=None, out=None, grads_out=None):
    """Forward AND backward of the same jagged batch (self-attention), the two
    running concurrently on two side streams after one band-table launch: the
    HSTU backward recomputes S and P from q, k, v (attention.py:187-234) and
    never reads the forward's output, so the forward's tail and the
    backward's head share the GPU (C2: ~2 % of the step).  Returns (out, dq,
    dk, dv, d_ts_weights); ``out`` / ``grads_out`` = preallocated bf16 tensors
    as in attn_fwd / attn_bwd(out=)."""
    dev = q.device
    nb = int(num_buckets)
    if nb > FUSED_NB_MAX:  # (the effective-bucket path syncs anyway: keep it simple)
        o = attn_fwd(q, k, v, ts, ts, q_offsets, num_heads, ts_weights, nb, out=out)
        g = attn_bwd(q, k, v, ts, ts, q_offsets, dout, num_heads, ts_weights, nb, seg_host=seg_host, out=grads_out)
        return (o,) + tuple(g[:4])
    if band_table is None:
        band_table = new_band_table(q.shape[0], q_offsets.numel() - 1, dev)
    main = torch.cuda.current_stream(dev)
    compute_band(q, ts, ts, q_offsets, num_heads, nb, band_table)
    key = (dev.index, main.cuda_stream)
    if key not in _FB_STREAMS:
        # the backward (the longer one) on a higher-priority stream and enqueued
        # first: its CTAs take the SMs, the forward's fill the backward's tail
        lo, hi = torch.cuda.Stream.priority_range()
        _FB_STREAMS[key] = (torch.cuda.Stream(dev, priority=lo), torch.cuda.Stream(dev, priority=hi))
    s_f, s_b = _FB_STREAMS[key]
    s_f.wait_stream(main)
    s_b.wait_stream(main)
    for t in (q, k, v, ts, q_offsets, dout, band_table):
        t.record_stream(s_f)
        t.record_stream(s_b)
    with torch.cuda.stream(s_b):
        dq, dk, dv, dw, _ = attn_bwd(q, k, v, ts, ts, q_offsets, dout, num_heads, ts_weights, nb, seg_host=seg_host,
                                     band_table=band_table, out=grads_out)
    with torch.cuda.stream(s_f):
        o = attn_fwd(q, k, v, ts, ts, q_offsets, num_heads, ts_weights, nb, out=out, band_table=band_table,
                     band_ready=True)
    main.wait_stream(s_f)
    main.wait_stream(s_b)
    for t in (o, dq, dk, dv, dw):
        t.record_stream(main)
    return o, dq, dk, dv, dw


# Backward variant.  None = auto: the two-kernel path (dK/dV kernel writes bf16
# dS tiles, the dQ GEMM reads them; fastest at C2) whenever its exact dS
# scratch fits the budget (ds_scratch_budget), else the same two kernels over
# kv windows with a bounded scratch (_attn_bwd_windowed), else -- no 128-wide
# window fits, or a positional bias -- the fused one-kernel path (dq reduced in
# fp32, O(L) memory).  True / False force the two-kernel / fused path.
DETERMINISTIC_DEFAULT = {"value": None}
_BWD_STATE: dict = {}


_TOTAL_MEM: dict = {}


def ds_scratch_budget(device) -> int:
    """Bytes the auto policy lets the dS scratch take: JH_DS_SCRATCH_BUDGET, or
    1/8 of what this process may allocate under its per-process memory
    fraction.  (Host-cheap on purpose: torch.cuda.memory_allocated builds the
    allocator's whole statistics dict, ~150 us per call.)"""
    import os
    env = os.environ.get("JH_DS_SCRATCH_BUDGET")
    if env:
        return int(float(env))
    dev = torch.device(device)
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _TOTAL_MEM:
        _TOTAL_MEM[key] = torch.cuda.get_device_properties(key).total_memory
    return int(_TOTAL_MEM[key] * torch.cuda.get_per_process_memory_fraction(key) // 8)


def ds_scratch_bytes(num_heads: int, q_offsets_host, q_pos0_host=None, kv_len_host=None, kv_start_host=None) -> int:
    """Exact dS scratch of the deterministic backward for host segment arrays
    (kv_start does not change it; accepted so seg_host tuples pass through)."""
    qo = np.ascontiguousarray(q_offsets_host, dtype=np.int64)
    qp = None if q_pos0_host is None else np.ascontiguousarray(q_pos0_host, dtype=np.int64)
    kl = None if kv_len_host is None else np.ascontiguousarray(kv_len_host, dtype=np.int64)
    vp = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    return int(_lib.lib().jh_attn_ds_scratch_bytes_segs(vp(qo), vp(qp), vp(kl), int(qo.size - 1), int(num_heads)))


def release_caches() -> None:
    """Drop the persistent per-device buffers (the fused backward's state) so a
    memory-capped measurement starts from what it allocates itself."""
    _BWD_STATE.clear()


def bwd_state(q_rows: int, num_segments: int, H: int, dp: int, device) -> torch.Tensor:
    """Persistent zero-initialised state of the fused backward (one per device
    and stream; every call leaves it zero again)."""
    need = int(_lib.lib().jh_attn_bwd_state_bytes(int(q_rows), int(num_segments), int(H), int(dp)))
    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    buf = _BWD_STATE.get(key)
    if buf is None or buf.numel() < need:
        buf = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=device)
        _BWD_STATE[key] = buf
    return buf


def attn_bwd(q, k, v, ts_q, ts_k, q_offsets, dout, num_heads, ts_weights, num_buckets=16, pos_weights=None,
             q_pos0=None, kv_start=None, kv_len=None, kv_len_total=None, accumulate_dkv=False, prof=None,
             max_kv_len=None, dq_accum=None, band_table=None, deterministic=None, dbg_count_buckets=False,
             seg_host=None, out=None, dkv_accum=None, _ds_buf=None):
    """Fused jagged HSTU backward (jh_attn_bwd).

    Returns (dq bf16, dk, dv, d_ts_weights f64, d_pos f64 or None); dk/dv are
    bf16, or fp32 accumulators when ``accumulate_dkv`` (CP partials); with
    ``dq_accum`` (fp32, q's shape) dq is added there and returned as dq;
    ``band_table`` filled by the forward call on the same inputs is reused
    (no recomputation).
    ``deterministic``: True = the two-kernel path over a bf16 dS scratch
    (bitwise reproducible dq; scratch ~H L^2 bytes per sequence), False = the
    fused kernel (dq reduced in fp32, O(L) memory), None = auto (the two-kernel
    path when its scratch fits ``ds_scratch_budget``, else kv windows of it,
    else the fused kernel).  ``seg_host`` =
    (q_offsets, q_pos0 or None, kv_len or None[, kv_start]) as host arrays sizes
    the scratch exactly (a segment-form call also needs kv_start there to be
    windowed); without it ``max_kv_len`` (>= every segment's q and kv
    length) gives a bound, and without either the lengths are read back from
    the device (one synchronisation).  ``out`` = (dq, dk, dv) bf16 tensors shaped
    like q (any 16-byte row stride, e.g. column views of one gradient buffer)
    to write into instead of allocating (not with dq_accum / accumulate_dkv or
    padded head dims).  ``dkv_accum`` = (dk, dv) fp32 tensors shaped like k (with
    ``accumulate_dkv``) to add the partials into instead of fresh zero buffers."""
    if deterministic is None:
        deterministic = DETERMINISTIC_DEFAULT["value"]
    w = ts_weights.to(device=q.device, dtype=torch.float32).contiguous()
    if int(num_buckets) > FUSED_NB_MAX:  # (see _effective_buckets) d_ts_weights padded back to num_buckets
        _check_weights(w, num_buckets)
        nb_eff = _effective_buckets(num_buckets, ts_q, ts_k)
        res = attn_bwd(q, k, v, ts_q, ts_k, q_offsets, dout, num_heads, w[:nb_eff].contiguous(), nb_eff,
                       pos_weights, q_pos0, kv_start, kv_len, kv_len_total, accumulate_dkv, prof, max_kv_len,
                       dq_accum, band_table, deterministic, dbg_count_buckets, seg_host, out, dkv_accum)
        d_w = torch.zeros(int(num_buckets), dtype=torch.float64, device=q.device)
        d_w[:nb_eff] = res[3]
        return res[0], res[1], res[2], d_w, res[4]
    pw = None if pos_weights is None else pos_weights.to(device=q.device, dtype=torch.float32).contiguous()
    H = int(num_heads)
    if q.dim() != 2 or q.shape[1] % H:
        raise ValueError(f"embed_dim {q.shape[-1]} not divisible by num_heads {H}")
    d = q.shape[1] // H
    dp = padded_head_dim(d)
    _require_cuda("dout", dout, torch.bfloat16)
    _rowmajor("dout", dout)
    qq, kk, vv, gg = (_pad_heads(t, H, d, dp) for t in (q, k, v, dout))
    a = _attn_args(qq, kk, vv, ts_q, ts_k, q_offsets, H, w, num_buckets, pw, q_pos0, kv_start, kv_len)
    a.score_scale = 1.0 / float(np.sqrt(d))
    a.dout, a.ld_do = gg.data_ptr(), gg.stride(0)
    if dq_accum is not None:
        if dq_accum.dtype != torch.float32 or dq_accum.shape != q.shape or dq_accum.stride(1) != 1:
            raise ValueError("dq_accum must be a float32 tensor shaped like q")
        dq = dq_accum
        dqk = _pad_heads(dq_accum, H, d, dp)
        a.dq_accum, a.ld_dq = dqk.data_ptr(), dqk.stride(0)
    elif out is not None:
        if dp != d or accumulate_dkv:
            raise ValueError("out= needs head_dim 64 or 128 and no accumulate_dkv")
        for name, t in zip(("dq", "dk", "dv"), out):
            _require_cuda(name, t, torch.bfloat16)
            _rowmajor(name, t)
            if t.shape != q.shape or (t.stride(0) * 2) % 16 or t.data_ptr() % 16:
                raise ValueError(f"{name} out must be shaped like q with 16-byte aligned rows")
        dq = dqk = out[0]
        a.dq, a.ld_dq = dqk.data_ptr(), dqk.stride(0)
    else:
        dq = torch.empty_like(q)
        dqk = dq if dp == d else torch.empty_like(qq)
        a.dq, a.ld_dq = dqk.data_ptr(), dqk.stride(0)
    if accumulate_dkv and dkv_accum is not None:
        dk, dv = dkv_accum
        for name, t in (("dk", dk), ("dv", dv)):
            if t.dtype != torch.float32 or tuple(t.shape) != tuple(kk.shape) or not t.is_contiguous():
                raise ValueError(f"dkv_accum {name} must be a contiguous float32 tensor shaped like k")
        a.dk_accum, a.dv_accum = dk.data_ptr(), dv.data_ptr()
        a.ld_dk = a.ld_dv = kk.shape[1]
    elif accumulate_dkv:
        dk = torch.zeros(kk.shape, dtype=torch.float32, device=k.device)
        dv = torch.zeros(vv.shape, dtype=torch.float32, device=v.device)
        a.dk_accum, a.dv_accum = dk.data_ptr(), dv.data_ptr()
        a.ld_dk = a.ld_dv = kk.shape[1]
    else:
        dk, dv = (out[1], out[2]) if out is not None else (torch.empty_like(kk), torch.empty_like(vv))
        a.dk, a.dv = dk.data_ptr(), dv.data_ptr()
        a.ld_dk, a.ld_dv = dk.stride(0), dv.stride(0)
    d_w = torch.zeros(num_buckets, dtype=torch.float64, device=q.device)
    a.d_ts_weights = d_w.data_ptr()
    d_pos = None
    if pw is not None:
        d_pos = torch.zeros(pw.numel(), dtype=torch.float64, device=q.device)
        a.d_pos_weights = d_pos.data_ptr()
    kvt = q.shape[0] if kv_len_total is None else kv_len_total
    ws, nbytes = _workspace(q.shape[0], kvt, a.num_segments, H, dp, q.device)
    a.workspace, a.workspace_bytes = ws.data_ptr(), nbytes
    if dbg_count_buckets:
        if deterministic:
            raise ValueError("dbg_count_buckets is a fused-backward debug mode")
        deterministic = False
    ds_bytes = None
    if deterministic is not False:
        if seg_host is not None:
            ds_bytes = ds_scratch_bytes(H, *seg_host)
        else:
            if max_kv_len is None:
                if a.num_segments == 0:
                    max_kv_len = 0
                else:
                    ql = int((q_offsets[1:] - q_offsets[:-1]).max().item())
                    max_kv_len = max(ql, int(kv_len.max().item())) if kv_len is not None else ql
            ds_bytes = int(_lib.lib().jh_attn_ds_scratch_bytes(kvt, a.num_segments, H, int(max_kv_len)))
        if deterministic is None:
            budget = ds_scratch_budget(q.device)
            deterministic = ds_bytes <= budget
            plain = q_pos0 is None and kv_start is None and kv_len is None
            segform_host = seg_host is not None and len(seg_host) >= 4 and all(x is not None for x in seg_host[:4])
            if (not deterministic and pw is None and dp == d and WINDOWED_BWD["enabled"]
                    and (plain or segform_host) and not (out is not None and not plain)):
                if plain:
                    qo_host = (np.asarray(seg_host[0], dtype=np.int64) if seg_host is not None
                               else q_offsets.cpu().numpy().astype(np.int64))
                    lens = np.diff(qo_host)
                    segs = (qo_host, np.zeros_like(lens), lens, qo_host[:-1].copy())
                    if seg_host is None:  # the bound was loose: size the scratch exactly
                        ds_bytes = ds_scratch_bytes(H, qo_host)
                        deterministic = ds_bytes <= budget
                else:
                    segs = tuple(np.asarray(x, dtype=np.int64) for x in (seg_host[0], seg_host[1], seg_host[2],
                                                                          seg_host[3]))
                if not deterministic:
                    extra = 0 if dq_accum is not None else 4 * q.numel()
                    win = _windowed_plan(segs, H, budget, q.device, extra)
                    if win is not None:
                        res = _attn_bwd_windowed(q, k, v, ts_q, ts_k, dout, H, w, num_buckets, segs, win, out,
                                                 prof, dq_accum, accumulate_dkv, dkv_accum, unique_kv=plain)
                        if res is not None:
                            return res
                        # (its buffers did not fit: the fused kernel below, O(L) memory)
    a.deterministic = int(bool(deterministic))
    a.dbg_count_buckets = int(bool(dbg_count_buckets))
    if deterministic:
        if _ds_buf is not None and _ds_buf.numel() >= ds_bytes:  # (the windowed path's preallocated scratch)
            ds = _ds_buf
        else:
            ds = torch.empty(ds_bytes, dtype=torch.uint8, device=q.device)
        a.ds_scratch, a.ds_scratch_bytes = ds.data_ptr(), ds_bytes
    else:
        st = bwd_state(q.shape[0], a.num_segments, H, dp, q.device)
        a.bwd_state, a.bwd_state_bytes = st.data_ptr(), st.numel()
    _band(a, band_table, ready=True)
    _prof(a, prof)
    check(_lib.lib().jh_attn_bwd(ctypes.byref(a), _stream(q)), "hstu_attention backward")
    if deterministic:
        _bump(3 if (pw is not None or band_table is not None) else 4)  # (band table) + build + dK/dV + dQ
    else:
        _bump(2 if (pw is not None or band_table is not None) else 3)  # (band table) + build + fused
    if dp != d:
        if dq_accum is not None:
            dq_accum.copy_(_unpad_heads(dqk, H, d, dp))
        else:
            dq.copy_(_unpad_heads(dqk, H, d, dp))
        dk, dv = _unpad_heads(dk, H, d, dp), _unpad_heads(dv, H, d, dp)
    return dq, dk, dv, d_w, d_pos


# Long-sequence backward when the whole-sequence dS scratch exceeds the budget:
# the two-kernel path over kv WINDOWS of width W (multiple of 128).  Call w
# covers kv rows [wW, (w+1)W) of every sequence against the q rows [wW, L) that
# see them, split into chunks of WINDOW_Q_CHUNK rows so the dK/dV kernel has
# enough items: segment-form calls (q_pos0 / kv_start / kv_len, the mode of the
# CP remote calls) over a compact copy of the window's K / V / timestamps, dq
# accumulated in fp32 across calls, dK / dV complete within their call (every q
# row that sees a window is in that call) and scattered back as bf16.  Extra
# memory: dq in fp32 (as the fused kernel's state) + the window's scratch
# (~2 H W sum(L) bytes, within the budget) + O(W B) for the window copies.  The
# tiles run at the two-kernel rate (~750 TF/s at long L vs ~520 for the fused
# kernel, profiles/r2_ncu_summary.md).
WINDOWED_BWD = {"enabled": True, "calls": 0}  # calls: completed windowed backward calls
WINDOW_Q_CHUNK = 16384


def _windowed_plan(segs, H: int, budget: int, device, dq_bytes: int = 0):
    """Window width W for _attn_bwd_windowed, or None (no width >= 128 fits).
    ``segs`` = host (q_offsets, q_pos0, kv_len, kv_start)."""
    qo = segs[0]
    rows = int(qo[-1] - qo[0])
    if rows == 0:
        return None
    # headroom: at most a quarter of what the process may still allocate (this
    # branch runs only for long sequences, where the allocator query is cheap
    # next to the backward itself)
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    cap = _TOTAL_MEM.get(idx) or torch.cuda.get_device_properties(idx).total_memory
    avail = cap * torch.cuda.get_per_process_memory_fraction(idx) - torch.cuda.memory_allocated(idx)
    budget = min(budget, int(avail - dq_bytes) // 4)
    # scratch of one call <= (rows + 64 per segment) * W * H * 2 bytes (64 x 128 bf16 blocks)
    nseg_bound = int(sum((int(n) + WINDOW_Q_CHUNK - 1) // WINDOW_Q_CHUNK + 1 for n in np.diff(qo)))
    W = budget // (2 * H * (rows + 64 * nseg_bound)) // 128 * 128
    W = min(W, 1 << 16)
    return W if W >= 128 else None


def window_segments(segs, W: int, q_chunk: int) -> list:
    """The windowed backward's decomposition (host, no GPU): for each kv window
    w = positions [wW, (w+1)W) of every segment, the segment arrays of one
    segment-form call -- (q_offsets, q_pos0, kv_len, host block, compact kv
    rows) where the host block is [q_offsets, q_pos0, kv_start, kv_len, kv row
    indices of the compact window copy].  ``segs`` = host (q_offsets, q_pos0,
    kv_len, kv_start) of the original call.  Every visible (q, kv) pair of the
    original call appears in exactly one window call (tests/test_windows.py)."""
    qo, qp, kl, ks = segs
    out = []
    nwin = int((int(kl.max(initial=0)) + W - 1) // W)
    for wi in range(nwin):
        w0 = wi * W
        o, qpn, ksn, kln, rows = [int(qo[0])], [], [], [], []
        c = 0  # compact kv row of the next window copy
        for s in range(qp.size):
            a, b, p0, n = int(qo[s]), int(qo[s + 1]), int(qp[s]), int(kl[s])
            i0 = max(0, w0 - p0)  # first q row whose position reaches the window
            if n <= w0 or a + i0 >= b:  # this segment has nothing in the window: one empty segment
                o.append(b); qpn.append(0); ksn.append(0); kln.append(0)
                continue
            if i0 > 0:  # rows before the window: empty segment
                o.append(a + i0); qpn.append(0); ksn.append(0); kln.append(0)
            wl = min(W, n - w0)
            for c0 in range(a + i0, b, q_chunk):
                o.append(min(b, c0 + q_chunk)); qpn.append(p0 + (c0 - a) - w0); ksn.append(c); kln.append(wl)
            rows.append(np.arange(int(ks[s]) + w0, int(ks[s]) + w0 + wl, dtype=np.int64))
            c += wl
        if c == 0:
            continue
        o_a, qp_a, kl_a = (np.asarray(x, dtype=np.int64) for x in (o, qpn, kln))
        host = np.concatenate([o_a, qp_a, np.asarray(ksn, dtype=np.int64), kl_a] + rows)
        out.append((o_a, qp_a, kl_a, host, c))
    return out


def _attn_bwd_windowed(q, k, v, ts_q, ts_k, dout, H, w, num_buckets, segs, W, out, prof, dq_accum=None,
                       accumulate_dkv=False, dkv_accum=None, unique_kv=False):
    """Segment s: q rows [qo[s], qo[s+1]) at positions qp[s] + i against kv rows
    ks[s] + j, j < kl[s] (kernels.attn_bwd's segment form; plain self-attention
    is qp = 0, ks = qo, kl = lengths).  Window w = kv positions [wW, (w+1)W): the
    q rows with position >= wW see it, in chunks of WINDOW_Q_CHUNK rows.  Every
    window is planned first and the scratch / window buffers are allocated
    once at their maximum: if they do not fit, None is returned before anything
    was accumulated (the caller then runs the fused kernel)."""
    dev = q.device
    wins = [w_ + (ds_scratch_bytes(H, w_[0], w_[1], w_[2]),) for w_ in window_segments(segs, W, WINDOW_Q_CHUNK)]
    if not wins:
        return None
    max_c = max(x[4] for x in wins)
    max_ds = max(x[5] for x in wins)
    try:
        ds_buf = torch.empty(max(max_ds, 1), dtype=torch.uint8, device=dev)
        kvw = torch.empty((2, max_c, k.shape[1]), dtype=k.dtype, device=dev)
        tsw = torch.empty(max_c, dtype=ts_k.dtype, device=dev)
        dkvw = torch.empty((2, max_c, k.shape[1]), dtype=torch.float32, device=dev)
        dq32 = dq_accum if dq_accum is not None else torch.zeros(q.shape, dtype=torch.float32, device=dev)
        if accumulate_dkv or not unique_kv:
            if dkv_accum is not None:
                dk32, dv32 = dkv_accum
            else:
                dk32 = torch.zeros(k.shape, dtype=torch.float32, device=dev)
                dv32 = torch.zeros(v.shape, dtype=torch.float32, device=dev)
            dk = dv = None
        else:  # every kv row belongs to one (segment, window): written once, as bf16
            dk32 = dv32 = None
            if out is not None:
                dk, dv = out[1], out[2]
            else:
                dk, dv = torch.empty_like(k), torch.empty_like(v)
    except torch.OutOfMemoryError:
        return None
    d_w = torch.zeros(num_buckets, dtype=torch.float64, device=dev)
    for o_a, qp_a, kl_a, host, c, _ in wins:
        m = qp_a.size
        # (pinned + non-blocking: a pageable copy would make the host wait for the
        # previous window's kernels before it can queue this one's)
        t = torch.from_numpy(host).pin_memory().to(dev, non_blocking=True)
        idx = t[4 * m + 1:]
        k_w, v_w, ts_w = kvw[0, :c], kvw[1, :c], tsw[:c]
        torch.index_select(k, 0, idx, out=k_w)
        torch.index_select(v, 0, idx, out=v_w)
        torch.index_select(ts_k, 0, idx, out=ts_w)
        dk_w, dv_w = dkvw[0, :c], dkvw[1, :c]
        dkvw[:, :c].zero_()
        # (q rows outside [o[0], o[-1]) belong to no segment of this call: the kernels never touch them)
        _, _, _, dwi, _ = attn_bwd(q, k_w, v_w, ts_q, ts_w, t[:m + 1], dout, H, w, num_buckets,
                                   q_pos0=t[m + 1:2 * m + 1], kv_start=t[2 * m + 1:3 * m + 1],
                                   kv_len=t[3 * m + 1:4 * m + 1], kv_len_total=c, accumulate_dkv=True,
                                   dkv_accum=(dk_w, dv_w), dq_accum=dq32, deterministic=True,
                                   seg_host=(o_a, qp_a, kl_a), prof=prof, _ds_buf=ds_buf)
        if dk32 is not None:
            dk32.index_add_(0, idx, dk_w)
            dv32.index_add_(0, idx, dv_w)
        else:
            dk.index_copy_(0, idx, dk_w.to(dk.dtype))
            dv.index_copy_(0, idx, dv_w.to(dv.dtype))
        d_w += dwi
    del ds_buf, kvw, tsw, dkvw
    WINDOWED_BWD["calls"] += 1
    if dk32 is not None and not accumulate_dkv:
        dk, dv = dk32.to(torch.bfloat16), dv32.to(torch.bfloat16)
        if out is not None:
            out[1].copy_(dk)
            out[2].copy_(dv)
            dk, dv = out[1], out[2]
    elif dk32 is not None:
        dk, dv = dk32, dv32
    if dq_accum is not None:
        return dq_accum, dk, dv, d_w, None
    if out is not None:
        out[0].copy_(dq32)
        return out[0], dk, dv, d_w, None
    return dq32.to(torch.bfloat16), dk, dv, d_w, None


def debug_umma(a: torch.Tensor, b: torch.Tensor, a_mode: int, b_mode: int) -> torch.Tensor:
    _require_cuda("a", a, torch.bfloat16)
    d = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    check(_lib.lib().jh_debug_umma(_ptr(a.contiguous()), _ptr(b.contiguous()), _ptr(d), a_mode, b_mode, _stream(a)),
          "debug_umma")
    return d


# ------------------------------------------------------- HSTU layer row work

def _ld(name, t, n):
    if t.dim() != 2 or t.stride(1) != 1 or t.shape[1] != n:
        raise ValueError(f"{name} must be 2-D [rows, {n}] with unit column stride")
    return t.stride(0)


def silu(x: torch.Tensor) -> torch.Tensor:
    """y = x sigmoid(x) (bf16, jh_silu_fwd)."""
    _require_cuda("x", x, torch.bfloat16)
    x = x.contiguous()
    y = torch.empty_like(x)
    check(_lib.lib().jh_silu_fwd(_ptr(x), _ptr(y), x.numel(), _stream(x)), "silu")
    _bump()
    return y


def silu_bwd(x: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
    _require_cuda("x", x, torch.bfloat16)
    _require_cuda("dy", dy, torch.bfloat16)
    x, dy = x.contiguous(), dy.contiguous()
    dx = torch.empty_like(x)
    check(_lib.lib().jh_silu_bwd(_ptr(x), _ptr(dy), _ptr(dx), x.numel(), _stream(x)), "silu_bwd")
    _bump()
    return dx


def _colsum_ws(rows: int, n: int, device):
    nb = int(_lib.lib().jh_colsum_workspace_bytes(rows, n))
    return torch.empty(nb, dtype=torch.uint8, device=device), nb


def silu_bwd_colsum(x: torch.Tensor, dy: torch.Tensor, dbias: torch.Tensor | None = None):
    """(dx, dbias): dx = silu'(x) dy and dbias (fp32 [n], added into when given)
    = column sums of dx -- the bias gradient of uvqk = SiLU(xn W + b) in the
    same pass (jh_silu_bwd_colsum)."""
    _require_cuda("x", x, torch.bfloat16)
    _require_cuda("dy", dy, torch.bfloat16)
    x, dy = x.contiguous(), dy.contiguous()
    rows, n = x.shape
    dx = torch.empty_like(x)
    if dbias is None:
        dbias = torch.zeros(n, dtype=torch.float32, device=x.device)
    ws, nb = _colsum_ws(rows, n, x.device)
    check(_lib.lib().jh_silu_bwd_colsum(_ptr(x), _ptr(dy), _ptr(dx), rows, n, _ptr(dbias), _ptr(ws), nb, _stream(x)),
          "silu_bwd_colsum")
    _bump(2)
    return dx, dbias


def colsum(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """fp32 column sums of a bf16 [rows, n] matrix (jh_colsum; added into ``out``)."""
    _require_cuda("x", x, torch.bfloat16)
    rows, n = x.shape
    ld = _ld("x", x, n)
    if out is None:
        out = torch.zeros(n, dtype=torch.float32, device=x.device)
    ws, nb = _colsum_ws(rows, n, x.device)
    check(_lib.lib().jh_colsum(_ptr(x), ld, rows, n, _ptr(out), _ptr(ws), nb, _stream(x)), "colsum")
    _bump(2)
    return out


def norm_gate_fwd(x, u=None, gamma=None, beta=None, eps: float = 1e-6):
    """y = (LayerNorm(x) * gamma + beta) * u per row (jh_norm_gate_fwd).
    x: [rows, n] bf16; u: [rows, n] bf16 view (any 16-B row stride) or None;
    gamma / beta: fp32 [n] or None.  Returns (y bf16, mean fp32, rstd fp32)."""
    _require_cuda("x", x, torch.bfloat16)
    rows, n = x.shape
    ldx = _ld("x", x, n)
    ldu = 0
    if u is not None:
        _require_cuda("u", u, torch.bfloat16)
        ldu = _ld("u", u, n)
    y = torch.empty((rows, n), dtype=torch.bfloat16, device=x.device)
    mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    g = None if gamma is None else gamma.to(device=x.device, dtype=torch.float32).contiguous()
    b = None if beta is None else beta.to(device=x.device, dtype=torch.float32).contiguous()
    check(_lib.lib().jh_norm_gate_fwd(_ptr(x), ldx, _ptr(u), ldu, _ptr(g), _ptr(b), float(eps), rows, n, _ptr(y), n,
                                      _ptr(mean), _ptr(rstd), _stream(x)), "norm_gate_fwd")
    _bump()
    return y, mean, rstd


def norm_gate_bwd(dy, x, u, gamma, beta, mean, rstd, need_affine: bool = True, du_out=None):
    """Gradients of norm_gate_fwd: (dx, du or None, dgamma or None, dbeta or None);
    ``du_out`` (bf16 [rows, n], any 16-byte row stride) receives du in place."""
    _require_cuda("dy", dy, torch.bfloat16)
    rows, n = x.shape
    dy = dy.contiguous()
    ldx = _ld("x", x, n)
    ldu = 0 if u is None else _ld("u", u, n)
    dx = torch.empty((rows, n), dtype=torch.bfloat16, device=x.device)
    du = None if u is None else (du_out if du_out is not None else
                                 torch.empty((rows, n), dtype=torch.bfloat16, device=x.device))
    lddu = n if du is None else _ld("du", du, n)
    g = None if gamma is None else gamma.to(device=x.device, dtype=torch.float32).contiguous()
    b = None if beta is None else beta.to(device=x.device, dtype=torch.float32).contiguous()
    dg = torch.zeros(n, dtype=torch.float32, device=x.device) if (need_affine and gamma is not None) else None
    db = torch.zeros(n, dtype=torch.float32, device=x.device) if (need_affine and beta is not None) else None
    ws, wsb = None, 0
    if dg is not None or db is not None:
        wsb = int(_lib.lib().jh_norm_gate_bwd_workspace_bytes(rows, n))
        ws = torch.empty(wsb, dtype=torch.uint8, device=x.device)
    check(_lib.lib().jh_norm_gate_bwd(_ptr(dy), n, _ptr(x), ldx, _ptr(u), ldu, _ptr(g), _ptr(b), _ptr(mean),
                                      _ptr(rstd), rows, n, _ptr(dx), n, _ptr(du), lddu, _ptr(dg), _ptr(db), _ptr(ws),
                                      wsb, _stream(x)), "norm_gate_bwd")
    _bump(2 if ws is not None else 1)
    return dx, du, dg, db
