"""ctypes binding of the C ABI ``include/jh_hstu.h`` (libjh_hstu.so).

This is the reference-side binding a maintainer of ``jaggedcp`` would add
(see INTEGRATION.md): plain pointers and sizes, no torch types cross the
ABI.  Loading fails loudly when the library is missing -- there is no CPU
fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libjh_hstu.so")

JH_OK, JH_ERR_INVALID, JH_ERR_CUDA, JH_ERR_UNSUPPORTED = 0, 1, 2, 3

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_vp = ctypes.c_void_p


class JhAttnArgs(ctypes.Structure):
    """Mirror of ``jh_attn_args`` (include/jh_hstu.h)."""

    _fields_ = [
        ("q", c_vp), ("k", c_vp), ("v", c_vp),
        ("ld_q", ctypes.c_int64), ("ld_k", ctypes.c_int64), ("ld_v", ctypes.c_int64),
        ("ts_q", c_vp), ("ts_k", c_vp),
        ("q_offsets", c_vp), ("q_pos0", c_vp), ("kv_start", c_vp), ("kv_len", c_vp),
        ("num_segments", ctypes.c_int64), ("q_rows", ctypes.c_int64), ("kv_rows", ctypes.c_int64),
        ("num_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("ts_weights", c_vp), ("num_buckets", ctypes.c_int32),
        ("pos_weights", c_vp), ("num_pos", ctypes.c_int32),
        ("max_q_len_hint", ctypes.c_int32),
        ("out", c_vp), ("ld_o", ctypes.c_int64),
        ("dout", c_vp), ("ld_do", ctypes.c_int64),
        ("dq", c_vp), ("dk", c_vp), ("dv", c_vp),
        ("ld_dq", ctypes.c_int64), ("ld_dk", ctypes.c_int64), ("ld_dv", ctypes.c_int64),
        ("dk_accum", c_vp), ("dv_accum", c_vp),
        ("d_ts_weights", c_vp), ("d_pos_weights", c_vp),
        ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t),
        ("prof_event_start", c_vp), ("prof_event_end", c_vp),
        ("trace", c_vp), ("trace_cta", ctypes.c_int32),
        ("ds_scratch", c_vp), ("ds_scratch_bytes", ctypes.c_size_t),
        ("out_accum", c_vp), ("out_accum_mode", ctypes.c_int32),
        ("dq_accum", c_vp),
        ("band_table", c_vp), ("band_table_bytes", ctypes.c_size_t), ("band_table_ready", ctypes.c_int32),
        ("score_scale", ctypes.c_float), ("deterministic", ctypes.c_int32),
        ("bwd_state", c_vp), ("bwd_state_bytes", ctypes.c_size_t),
        ("dbg_buckets", c_vp), ("dbg_ld", ctypes.c_int64), ("dbg_count_buckets", ctypes.c_int32),
    ]


# name -> (restype, argtypes); every symbol include/jh_hstu.h declares
SIGNATURES = {
    "jh_last_error": (ctypes.c_char_p, []),
    "jh_version": (ctypes.c_int, []),
    "jh_bias_table_build": (ctypes.c_int, [ctypes.c_int, c_i64p, c_i32p, c_i64p]),
    "jh_bucketize": (ctypes.c_int, [c_vp, ctypes.c_int64, ctypes.c_int, c_vp, c_vp]),
    "jh_compute_bias": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, c_vp, ctypes.c_int, c_vp, c_vp]),
    "jh_dbias_scatter": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, c_vp, ctypes.c_int, c_vp, c_vp]),
    "jh_attn_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                                  ctypes.c_int32]),
    "jh_attn_band_table_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64]),
    "jh_attn_ds_scratch_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64]),
    "jh_attn_ds_scratch_bytes_segs": (ctypes.c_size_t, [c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int32]),
    "jh_attn_bwd_state_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]),
    "jh_silu_fwd": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, c_vp]),
    "jh_silu_bwd": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int64, c_vp]),
    "jh_silu_bwd_colsum": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int32, c_vp, c_vp,
                                          ctypes.c_size_t, c_vp]),
    "jh_colsum": (ctypes.c_int, [c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, c_vp, c_vp, ctypes.c_size_t,
                                 c_vp]),
    "jh_colsum_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32]),
    "jh_norm_gate_fwd": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, c_vp, c_vp, ctypes.c_float,
                                        ctypes.c_int64, ctypes.c_int32, c_vp, ctypes.c_int64, c_vp, c_vp, c_vp]),
    "jh_norm_gate_bwd_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32]),
    "jh_norm_gate_bwd": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, c_vp, c_vp,
                                        c_vp, c_vp, ctypes.c_int64, ctypes.c_int32, c_vp, ctypes.c_int64, c_vp,
                                        ctypes.c_int64, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp]),
    "jh_attn_fwd": (ctypes.c_int, [ctypes.POINTER(JhAttnArgs), c_vp]),
    "jh_attn_band": (ctypes.c_int, [ctypes.POINTER(JhAttnArgs), c_vp]),
    "jh_attn_bwd": (ctypes.c_int, [ctypes.POINTER(JhAttnArgs), c_vp]),
    "jh_gather_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, c_vp]),
    "jh_scatter_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, c_vp]),
    "jh_jagged_to_padded": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, c_vp, c_vp]),
    "jh_padded_to_jagged": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, c_vp, c_vp]),
    "jh_plan_build": (ctypes.c_int, [c_i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, c_i64p, c_i64p, c_i32p]),
    "jh_flops_per_rank": (ctypes.c_int, [c_i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, c_i64p, c_i64p]),
    "jh_rank_major_perm": (ctypes.c_int, [c_i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, c_i64p, c_i64p]),
    "jh_debug_umma": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_vp]),
}

_lib = None


class JhError(RuntimeError):
    pass


def lib():
    """Load libjh_hstu.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -C paper_2508_04711_b200/csrc).  There is no CPU fallback."
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    """Map a jh status code to the reference's exception types."""
    if rc == JH_OK:
        return
    msg = lib().jh_last_error().decode(errors="replace")
    if rc == JH_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    if rc == JH_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise JhError(f"{what}: {msg}")
