"""GPU parity of the fused jagged HSTU attention against the CPU oracle.

Tolerance (bf16 inputs, fp32 accumulation, bf16 P and outputs): the
reference's own row-normalized error metric (harness.py:189-206,
||got-want||_inf,row / max(1, ||want||_inf,row)) <= 2e-2 for out/dq/dk/dv,
and max|d_w - ref| / max|ref| <= 1e-3 for d_ts_weights.  The oracle is fed
the identical bf16-rounded inputs (f32 arithmetic).
"""

import os

import numpy as np
import pytest
import torch

import oracle
from _cases import make_case, synthetic, to_cuda, row_rel
from conftest import load_npz_cases

pytestmark = pytest.mark.gpu

ROW_TOL = 1e-2  # measured 3-7e-3 (bf16 P / dS / outputs, L <= 1024); 2e-2 before round 2
ROW_TOL_LONG = 1e-2  # L up to 4096 (error grows slowly with L: 3-6e-3 measured)
DW_TOL = 1e-3


def _fwd(case, H, pos=None):
    from paper_2508_04711_b200 import kernels
    c = to_cuda(case)
    out = kernels.attn_fwd(c["q"], c["k"], c["v"], c["ts"], c["ts"], c["offsets"], H, c["w"], case["nb"],
                           pos_weights=None if pos is None else torch.from_numpy(pos).float().cuda())
    torch.cuda.synchronize()
    return out.float().cpu().numpy()


@pytest.mark.parametrize("lens,H,d", [
    ([1], 1, 128), ([5, 0, 17, 1, 32], 1, 64), ([128], 1, 128), ([129, 255, 256, 257], 2, 64),
    ([300, 77, 1000], 4, 128), ([513, 1, 2, 3], 2, 128),
])
def test_fwd_matches_oracle(lens, H, d):
    case = make_case(lens, H * d, seed=sum(lens) + H)
    got = _fwd(case, H)
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, H)
    _, rel = row_rel(got, want)
    assert rel <= ROW_TOL, rel


def test_fwd_unsorted_timestamps_and_small_gaps():
    # exercises the per-element bucket path on every tile (no saturation)
    case = make_case([400, 200], 128, seed=5, unsorted_ts=True)
    got = _fwd(case, 1)
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, 1)
    assert row_rel(got, want)[1] <= ROW_TOL


@pytest.mark.parametrize("name", ["f32_c1_bf16", "f32_d64_bf16_long"])
def test_fwd_matches_reference_golden(name):
    c = load_npz_cases("attention_cases.npz")[name]
    H, nb = (int(x) for x in c["meta"])
    case = dict(q=c["q"], k=c["k"], v=c["v"], ts=c["ts"], offsets=c["offsets"], w=c["w"], nb=nb)
    got = _fwd(case, H)
    assert row_rel(got, c["o"])[1] <= ROW_TOL


def test_fwd_synthetic_c2_subset():
    b = synthetic(7, 0, 8, 1024, 4, 128)
    case = dict(q=b["q"], k=b["k"], v=b["v"], ts=b["ts"], offsets=b["offsets"],
                w=oracle.normal_init_ts_weights(16, 7 + 0x5EED), nb=16)
    got = _fwd(case, 4)
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, 4)
    assert row_rel(got, want)[1] <= ROW_TOL


def _bwd(case, H, pos=None, det=False):
    from paper_2508_04711_b200 import kernels
    c = to_cuda(case)
    dq, dk, dv, dw, dpos = kernels.attn_bwd(
        c["q"], c["k"], c["v"], c["ts"], c["ts"], c["offsets"], c["g"], H, c["w"], case["nb"],
        pos_weights=None if pos is None else torch.from_numpy(pos).float().cuda(), deterministic=det)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    return f(dq), f(dk), f(dv), dw.cpu().numpy(), None if dpos is None else dpos.cpu().numpy()


def _check_bwd(case, H, got, tol=ROW_TOL):
    dq, dk, dv, dw, _ = got
    wq, wk, wv, ww, _ = oracle.hstu_backward(case["q"], case["k"], case["v"], case["ts"], case["offsets"],
                                              case["g"], case["w"], case["nb"], H)
    for name, a, b in (("dq", dq, wq), ("dk", dk, wk), ("dv", dv, wv)):
        mx, rel = row_rel(a, b)
        print(f"{name}: max_abs={mx:.3e} row_rel={rel:.3e}")
        assert rel <= tol, (name, mx, rel)
    assert np.abs(dw - ww).max() / max(np.abs(ww).max(), 1e-30) <= DW_TOL, (dw, ww)


@pytest.mark.parametrize("lens,H,d", [
    ([1], 1, 128), ([5, 0, 17, 1, 32], 1, 64), ([128], 1, 128), ([129, 255, 256, 257], 2, 64),
    ([300, 77, 1000], 4, 128), ([513, 1, 2, 3], 2, 128),
])
@pytest.mark.parametrize("det", [False, True], ids=["fused", "deterministic"])
def test_bwd_matches_oracle(lens, H, d, det):
    case = make_case(lens, H * d, seed=sum(lens) + 7 * H)
    _check_bwd(case, H, _bwd(case, H, det=det))


@pytest.mark.parametrize("det", [False, True], ids=["fused", "deterministic"])
def test_bwd_unsorted_timestamps(det):
    case = make_case([400, 200], 128, seed=5, unsorted_ts=True)
    _check_bwd(case, 1, _bwd(case, 1, det=det))


@pytest.mark.parametrize("name", ["f32_c1_bf16", "f32_d64_bf16_long"])
def test_bwd_matches_reference_golden(name):
    c = load_npz_cases("attention_cases.npz")[name]
    H, nb = (int(x) for x in c["meta"])
    case = dict(q=c["q"], k=c["k"], v=c["v"], g=c["g"], ts=c["ts"], offsets=c["offsets"], w=c["w"], nb=nb)
    dq, dk, dv, dw, _ = _bwd(case, H)
    for a, b in ((dq, c["dq"]), (dk, c["dk"]), (dv, c["dv"])):
        assert row_rel(a, b)[1] <= ROW_TOL
    assert np.abs(dw - c["dw"]).max() / np.abs(c["dw"]).max() <= DW_TOL


# ------------------------------------------------ timestamp regimes (band table)

def _ts_case(lens, D, gap_max, seed, equal=False):
    case = make_case(lens, D, seed=seed, ts_gap_max=max(gap_max, 1))
    if equal:  # every delta 0 -> bucket 0 for every pair: nothing saturates anywhere
        offs = case["offsets"]
        for b in range(len(lens)):
            case["ts"][offs[b]:offs[b + 1]] = 12345 + b
    return case


@pytest.mark.parametrize("gap_max,equal", [(1000, False), (1, True), (10**9, False), (30_000, False)])
def test_fwd_bwd_timestamp_regimes(gap_max, equal):
    # gaps << cap: unsaturated far beyond the band-table window (general path
    # outside it); equal timestamps: bucket 0 everywhere; huge gaps: saturated
    # right next to the diagonal; 30K: the band spans ~100 columns (window edge)
    H = 2
    case = _ts_case([700, 129, 1, 64, 333], H * 128, gap_max, seed=gap_max % 97 + int(equal), equal=equal)
    got = _fwd(case, H)
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, H)
    assert row_rel(got, want)[1] <= ROW_TOL
    _check_bwd(case, H, _bwd(case, H))
    _check_bwd(case, H, _bwd(case, H, det=True))


# ------------------------------------------------ full-size configs (sampled)

def test_c2_full_batch_matches_oracle():
    # the bench workload itself (BASELINE configs[1]): B=32, L<=1024, H=4, d=128,
    # bf16; every output row checked against the oracle, d_ts_weights over the batch
    b = synthetic(7, 0, 32, 1024, 4, 128)
    rng = np.random.default_rng(99)
    g = rng.standard_normal(b["q"].shape).astype(np.float32)
    from _cases import bf16_round
    case = dict(q=b["q"], k=b["k"], v=b["v"], g=bf16_round(g), ts=b["ts"], offsets=b["offsets"],
                w=oracle.normal_init_ts_weights(16, 7 + 0x5EED), nb=16)
    got = _fwd(case, 4)
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, 4)
    assert row_rel(got, want)[1] <= ROW_TOL
    _check_bwd(case, 4, _bwd(case, 4))
    _check_bwd(case, 4, _bwd(case, 4, det=True))


def test_long_sequences_c3_lengths():
    # C3-like lengths (up to 4096) with the reference generator's timestamps
    H = 2
    case = make_case([4096, 2500, 1], H * 128, seed=41)
    got = _fwd(case, H)
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, H)
    assert row_rel(got, want)[1] <= ROW_TOL_LONG
    _check_bwd(case, H, _bwd(case, H), tol=ROW_TOL_LONG)
    _check_bwd(case, H, _bwd(case, H, det=True), tol=ROW_TOL_LONG)


def test_two_tile_forward_variant_matches_oracle():
    # attn_fwd2.cu (two q tiles per K/V load, JH_FWD2=1; the library reads the
    # switch once per process, so the check runs in a child process)
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, oracle
from _cases import make_case, row_rel, to_cuda
from paper_2508_04711_b200 import kernels
for lens, H, d in (([300, 1, 0, 129, 64, 257], 2, 128), ([700, 33], 1, 64)):
    case = make_case(lens, H * d, seed=len(lens))
    c = to_cuda(case)
    out = kernels.attn_fwd(c["q"], c["k"], c["v"], c["ts"], c["ts"], c["offsets"], H, c["w"], 16)
    torch.cuda.synchronize()
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, H)
    err = row_rel(out.float().cpu().numpy(), want)[1]
    assert err <= 1e-2, err
print("ok")
"""
    env = dict(os.environ, JH_FWD2="1", PYTHONPATH=os.pathsep.join([os.path.dirname(__file__),
                                                                      os.path.dirname(os.path.dirname(__file__))]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
