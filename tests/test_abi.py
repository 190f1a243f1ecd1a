"""CPU checks of the C ABI: the library loads, exports every symbol the
header declares, and its host-side integer functions (bucket table, CP plan,
flop counts, rank-major permutation) are bit-exact with the oracle/reference."""

import ctypes
import json
import os
import re

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "jh_hstu.h")


@pytest.fixture(scope="module")
def L():
    from paper_2508_04711_b200 import _lib
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    from paper_2508_04711_b200 import _lib
    names = re.findall(r"JH_API\s+[\w\*\s]+?\b(jh_\w+)\s*\(", open(HEADER).read())
    assert len(names) >= 17
    for n in names:
        assert hasattr(L, n), n
        assert n in _lib.SIGNATURES, n


def _table_bucket(d, thr, base, cap):
    d = np.clip(np.asarray(d, dtype=np.int64), 0, cap)
    o = np.floor(np.log2((d + 1).astype(np.float64))).astype(np.int64)
    # exact octave via integer bit length (float log2 may round near 2^k)
    o = np.array([int(x + 1).bit_length() - 1 for x in d], dtype=np.int64)
    return base[o] + (d >= thr[o]).astype(np.int64)


@pytest.mark.parametrize("nb", [1, 2, 8, 16, 33, 40, 64])
def test_bucket_table_bit_exact_vs_reference(nb):
    from paper_2508_04711_b200 import kernels
    thr, base, cap = kernels.bias_table(nb)
    g = np.load(os.path.join(GOLDEN, "buckets.npz"))
    got = _table_bucket(g["deltas"], thr, base, cap)
    assert np.array_equal(got, g[f"nb{nb}"])


def test_bucket_table_exhaustive_small_range():
    from paper_2508_04711_b200 import kernels
    thr, base, cap = kernels.bias_table(16)
    d = np.arange(-100, 4_000_000, dtype=np.int64)
    assert np.array_equal(_table_bucket(d, thr, base, cap), oracle.bucketize_array(d, 16))


def _plan_via_abi(L, lengths, cp, mode):
    n = len(lengths)
    C = 2 * cp if mode == 0 else cp
    ln = (ctypes.c_int64 * max(n, 1))(*lengths)
    cl = (ctypes.c_int64 * max(n * C, 1))()
    cs = (ctypes.c_int64 * max(n * C, 1))()
    co = (ctypes.c_int32 * C)()
    assert L.jh_plan_build(ln, n, cp, mode, cl, cs, co) == 0
    return np.array(cl[: n * C]).reshape(n, C), np.array(cs[: n * C]).reshape(n, C), list(co)


def test_plan_matches_reference_fixture(L):
    rec = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for p in rec["plans"]:
        lens = [x for r in p["lengths_per_rank"] for x in r]
        mode = 0 if p["mode"] == "balanced_minichunk" else 1
        cl, cs, co = _plan_via_abi(L, lens, p["cp"], mode)
        assert co == p["chunk_owner"]
        assert cl.tolist() == p["chunk_lengths"]
        pr = (ctypes.c_int64 * p["cp"])()
        tot = ctypes.c_int64()
        ln = (ctypes.c_int64 * max(len(lens), 1))(*lens)
        assert L.jh_flops_per_rank(ln, len(lens), p["cp"], mode, pr, ctypes.byref(tot)) == 0
        assert list(pr) == p["flops_per_rank"] and tot.value == p["flops_total"]
        # rank entries: (seq, chunk, start, end) for chunks the rank owns, seq then chunk order
        for r in range(p["cp"]):
            ents = [[b, c, int(cs[b, c]), int(cs[b, c] + cl[b, c])]
                    for b in range(len(lens)) for c in range(len(co)) if co[c] == r]
            assert ents == p["rank_entries"][r]


def test_rank_major_perm_matches_reference(L):
    rec = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for r in rec["reorders"]:
        offs = np.concatenate([[0], np.cumsum(r["lengths"])]).astype(np.int64)
        T = int(offs[-1])
        perm = (ctypes.c_int64 * max(T, 1))()
        slab = (ctypes.c_int64 * r["cp"])()
        o = (ctypes.c_int64 * len(offs))(*offs.tolist())
        assert L.jh_rank_major_perm(o, len(offs) - 1, r["cp"], 0, perm, slab) == 0
        assert list(perm[:T]) == r["perm"]
        bounds = np.concatenate([[0], np.cumsum(list(slab))])
        assert [[int(bounds[i]), int(bounds[i + 1])] for i in range(r["cp"])] == r["rank_row_ranges"]


def test_plan_rejects_bad_args(L):
    ln = (ctypes.c_int64 * 1)(4)
    cl = (ctypes.c_int64 * 8)()
    cs = (ctypes.c_int64 * 8)()
    co = (ctypes.c_int32 * 8)()
    assert L.jh_plan_build(ln, 1, 0, 0, cl, cs, co) == 1
    assert b"cp_size" in L.jh_last_error()
    assert L.jh_plan_build(ln, 1, 2, 7, cl, cs, co) == 1
    assert b"balance_mode" in L.jh_last_error()


def _ds_cnt_py(lq, qp0, kvl):
    # attn_common.cuh ds_cnt, restated: causal triangle of (128-row kv tile, 64-row q half) blocks
    if lq <= 0:
        return 0
    vis = min(qp0 + lq, kvl)
    nkt = -(-vis // 128) if vis > 0 else 0
    nh = -(-lq // 64)
    m = -(-qp0 // 128)
    x = nkt - 1 - m
    cnt = nkt * nh - (x * (x + 1) if x >= 0 else 0)
    # brute force: blocks (j, t) with t >= tlo(j) = 2 * max(0, floor((128 j - qp0) / 128))
    brute = 0
    for j in range(nkt):
        f = 128 * j - qp0
        tlo = 0 if f <= 0 else (f // 128) * 2
        brute += max(nh - tlo, 0)
    assert cnt == brute
    return cnt


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ds_scratch_exact_and_bound(L, seed):
    # exact size = sum of the per-segment block counts; the bound (max_len >= q and
    # kv lengths) covers it, including CP "remote" segments with q longer than kv
    from paper_2508_04711_b200 import kernels
    rng = np.random.default_rng(seed)
    n = 12
    lq = rng.integers(0, 5000, n)
    qp0 = np.where(rng.random(n) < 0.5, 0, rng.integers(0, 6000, n))
    kvl = np.where(qp0 == 0, lq, rng.integers(1, 6000, n))
    qo = np.concatenate([[0], np.cumsum(lq)]).astype(np.int64)
    H = 3
    want = max(sum(_ds_cnt_py(int(a), int(b), int(c)) for a, b, c in zip(lq, qp0, kvl)), 1) * H * 16384
    assert kernels.ds_scratch_bytes(H, qo, qp0, kvl) == want
    bound = L.jh_attn_ds_scratch_bytes(int(kvl.sum()), n, H, int(max(lq.max(), kvl.max())))
    assert bound >= want
    # the ADVICE case: one 4096-token sequence at CP=1 in the remote form (q [2048, 4096) vs kv [0, 2048))
    one = kernels.ds_scratch_bytes(4, np.array([0, 2048]), np.array([2048]), np.array([2048]))
    assert one == 4 * 16 * 32 * 16384
    assert L.jh_attn_ds_scratch_bytes(2048, 1, 4, 2048) >= one


def test_attn_entry_points_validate_before_touching_the_gpu(L):
    # argument errors are reported through the status code / jh_last_error
    # before any CUDA call (runs without a GPU)
    from paper_2508_04711_b200._lib import JH_ERR_INVALID, JhAttnArgs
    a = JhAttnArgs()
    assert L.jh_attn_band(None, None) == JH_ERR_INVALID
    assert b"NULL" in L.jh_last_error()
    buf = (ctypes.c_int64 * 8)()
    a.q_offsets = a.ts_q = a.ts_k = ctypes.cast(buf, ctypes.c_void_p).value
    a.num_segments, a.q_rows, a.num_heads, a.num_buckets = 1, 64, 1, 16
    assert L.jh_attn_band(ctypes.byref(a), None) == JH_ERR_INVALID  # no band table
    assert b"band_table" in L.jh_last_error()
    a.num_buckets = 0
    assert L.jh_attn_band(ctypes.byref(a), None) == JH_ERR_INVALID
    a.num_buckets, a.num_pos = 16, 3  # a positional bias has no band table: nothing to do
    assert L.jh_attn_band(ctypes.byref(a), None) == 0
    a.num_pos, a.q_rows = 0, 0  # empty: nothing to do
    assert L.jh_attn_band(ctypes.byref(a), None) == 0
    # the layer's column sums: shape and workspace checks
    assert L.jh_colsum(None, 8, 4, 8, None, None, 0, None) == JH_ERR_INVALID
    assert L.jh_silu_bwd_colsum(None, None, None, 4, 8, None, None, 0, None) == JH_ERR_INVALID
    assert L.jh_colsum_workspace_bytes(1000, 512) >= 512 * 4
