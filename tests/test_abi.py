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
