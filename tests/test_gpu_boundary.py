"""GPU tests of the drop-in boundary: the reference-signature entry points
(attention.py:125/151/187, harness.py:270) against the CPU oracle, the
small-head-dim path (zero-padded to 64 columns, 1/sqrt(d) kept), and the
validation errors.

Tolerance: the reference's row-normalised metric (harness.py:189-206) <= ROW_TOL
for bf16 inputs with fp32 accumulation (measured ~3e-3); max-abs is printed.
"""

import os

import numpy as np
import pytest
import torch

import oracle
from _cases import bf16_round, make_case, row_rel
from conftest import load_npz_cases

pytestmark = pytest.mark.gpu

ROW_TOL = 1e-2  # measured 3-7e-3
DW_TOL = 1e-3


def _report(name, got, want):
    mx, rel = row_rel(got, want)
    print(f"{name}: max_abs={mx:.3e} row_rel={rel:.3e}")
    return rel


def test_blockwise_partial_reference_signature_golden():
    import paper_2508_04711_b200 as pkg
    c = load_npz_cases("blockwise_cases.npz")["b0"]
    q, k, v = (bf16_round(c[x].astype(np.float32)) for x in ("q", "k", "v"))
    params, cfg = pkg.BiasParams(c["w"]), pkg.BiasConfig(16)
    got = pkg.blockwise_partial(q, c["qs"], c["qp"], c["tq"], k, c["ks"], c["kp"], c["tk"], v, params, cfg)
    assert got.shape == c["out"].shape and got.dtype == torch.float32
    got = got.cpu().numpy()
    want = oracle.blockwise_partial(q.astype(np.float64), c["qs"], c["qp"], c["tq"], k.astype(np.float64), c["ks"],
                                    c["kp"], c["tk"], v.astype(np.float64), c["w"], 16)
    assert _report("blockwise(oracle)", got, want) <= ROW_TOL
    # the reference's own f64 output on the unrounded inputs (bf16 input rounding on top)
    assert _report("blockwise(golden)", got, c["out"]) <= 3e-2
    with pytest.raises(ValueError, match="rows but v has"):
        pkg.blockwise_partial(q, c["qs"], c["qp"], c["tq"], k, c["ks"], c["kp"], c["tk"], v[:3], params, cfg)
    z = pkg.blockwise_partial(q[:0], c["qs"][:0], c["qp"][:0], c["tq"][:0], k, c["ks"], c["kp"], c["tk"], v,
                              params, cfg)
    assert tuple(z.shape) == (0, 8)


@pytest.mark.parametrize("d,seed", [(128, 1), (64, 2), (8, 3)])
def test_blockwise_partial_cp_ring_blocks_sum_to_forward(d, seed):
    # block additivity (test_attention.py:220-250): partials over a partition of
    # the keys sum to the full forward
    import paper_2508_04711_b200 as pkg
    lens = [300, 77, 513]
    case = make_case(lens, d, seed=seed)
    offs = case["offsets"]
    seq = np.repeat(np.arange(len(lens)), lens)
    pos = np.concatenate([np.arange(L) for L in lens])
    params, cfg = pkg.BiasParams(case["w"]), pkg.BiasConfig(16)
    parts = np.array_split(np.random.default_rng(seed).permutation(int(offs[-1])), 3)
    total = 0
    for idx in parts:
        idx = np.sort(idx)
        total = total + pkg.blockwise_partial(case["q"], seq, pos, case["ts"], case["k"][idx], seq[idx], pos[idx],
                                              case["ts"][idx], case["v"][idx], params, cfg).cpu().numpy()
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], offs, case["w"], 16, 1)
    assert _report(f"blockwise sum d={d}", total, want) <= ROW_TOL


@pytest.mark.parametrize("lens,H,d", [([5, 0, 17, 33], 2, 8), ([130, 1, 64], 3, 32), ([200, 9], 1, 96)])
def test_small_head_dims_through_reference_api(lens, H, d):
    import paper_2508_04711_b200 as pkg
    case = make_case(lens, H * d, seed=sum(lens) + d)
    offs = case["offsets"]
    ml = max(max(lens), 1)
    J = lambda x: pkg.new_jagged(torch.from_numpy(x), offs, ml, device="cuda")  # noqa: E731
    inp = pkg.AttentionInputs(J(case["q"]), J(case["k"]), J(case["v"]),
                              pkg.new_int_series(case["ts"], offs, device="cuda"), pkg.BiasParams(case["w"]),
                              pkg.BiasConfig(16), num_heads=H)
    out = pkg.hstu_attention_reference(inp).values.float().cpu().numpy()
    want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], offs, case["w"], 16, H)
    assert _report(f"fwd d={d}", out, want) <= ROW_TOL
    gr = pkg.hstu_attention_backward(inp, J(case["g"]))
    wq, wk, wv, ww, _ = oracle.hstu_backward(case["q"], case["k"], case["v"], case["ts"], offs, case["g"], case["w"],
                                             16, H)
    for name, got, want in (("dq", gr.dq, wq), ("dk", gr.dk, wk), ("dv", gr.dv, wv)):
        assert _report(f"{name} d={d}", got.values.float().cpu().numpy(), want) <= ROW_TOL, name
    dw = gr.d_ts_weights.cpu().numpy()
    assert np.abs(dw - ww).max() <= DW_TOL * np.abs(ww).max()


def test_ts_weights_shorter_than_num_buckets_raises():
    from paper_2508_04711_b200 import kernels
    case = make_case([10], 64, seed=0)
    t = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    q = t(case["q"]).bfloat16()
    with pytest.raises(ValueError, match="num_buckets"):
        kernels.attn_fwd(q, q, q, t(case["ts"]), t(case["ts"]), t(case["offsets"]), 1,
                         torch.zeros(8, device="cuda"), 16)


def _oracle_reference(batches, params, bias_cfg, num_heads):
    """harness.py:173-186 on the CPU oracle (the bf16 values the GPU holds, upcast)."""
    vals = lambda b, f: getattr(b, f).values.float().cpu().numpy()  # noqa: E731
    cat = {f: np.concatenate([vals(b, f) for b in batches]) for f in ("q", "k", "v")}
    ts = np.concatenate([b.ts.values.cpu().numpy() for b in batches])
    offs = [0]
    for b in batches:
        base = offs[-1]
        offs.extend(int(base + o) for o in b.q.host_offsets[1:])
    out = oracle.hstu_forward(cat["q"], cat["k"], cat["v"], ts, np.asarray(offs), np.asarray(params.ts_weights),
                              bias_cfg.num_buckets, num_heads)
    res, row = [], 0
    for b in batches:
        n = int(b.q.host_offsets[-1])
        res.append(out[row:row + n])
        row += n
    return res


@pytest.mark.parametrize("cp,mode,sched", [(2, "balanced_minichunk", "sequential"),
                                           (4, "naive_contiguous", "threaded")])
def test_run_experiment_checked_against_oracle(cp, mode, sched):
    from paper_2508_04711_b200 import harness
    cfg = harness.ExperimentConfig(cp_size=cp, batch_size=3, min_len=0, max_len=300, max_length=512, embed_dim=128,
                                   num_heads=1, balance_mode=mode, seed=5)
    rep = harness.run_experiment(cfg, scheduling=sched, reference=_oracle_reference)
    print(f"run_experiment cp={cp}: max_abs={rep.max_abs_error:.3e} row_rel={rep.max_rel_error:.3e}")
    assert rep.max_rel_error <= ROW_TOL


# -------------------------------------------- reorder_balanced / inverse_reorder

@pytest.mark.parametrize("lens,cp,mode", [([4], 2, "balanced_minichunk"), ([300, 0, 17, 129], 3, "balanced_minichunk"),
                                          ([8, 5], 2, "naive_contiguous")])
def test_reorder_balanced_and_inverse_are_bitwise(lens, cp, mode):
    # jagged.py:232-258: rows in rank-major order (perm bit-exact with the
    # reference's _rank_major_row_order), values moved bitwise, exact inverse
    import oracle
    from paper_2508_04711_b200.jagged import (inverse_reorder, make_contiguous_chunks, make_minichunks,
                                              new_jagged, reorder_balanced)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    vals = torch.randn(T, 64, device="cuda").bfloat16()
    jt = new_jagged(vals, offs, max(lens))
    layout = make_minichunks(lens, cp) if mode == "balanced_minichunk" else make_contiguous_chunks(lens, cp)
    out, perm = reorder_balanced(jt, layout)
    from oracle.jagged import make_contiguous_chunks as o_contig, make_minichunks as o_mini
    olayout = o_mini(lens, cp) if mode == "balanced_minichunk" else o_contig(lens, cp)
    want_perm, _ = oracle.rank_major_row_order(offs, olayout)
    assert np.array_equal(perm.cpu().numpy(), np.asarray(want_perm))
    assert torch.equal(out.values, vals[perm])
    back = inverse_reorder(out, perm)
    assert torch.equal(back.values, vals)
    if lens == [4]:
        assert perm.cpu().tolist() == [0, 3, 1, 2]  # rank 0 owns chunks (0, 3), rank 1 (1, 2)
    with pytest.raises(ValueError, match="bijection"):
        inverse_reorder(out, torch.zeros(T, dtype=torch.int64))


def test_measured_sweep_small_budget():
    # harness.sweep_max_tokens_measured: the reference's SweepReport schema, lengths
    # non-decreasing in CP (one rank's share shrinks), a 2-layer stack under a 2 GB cap
    from paper_2508_04711_b200.harness import sweep_max_tokens_measured
    rep = sweep_max_tokens_measured(int(2e9), (1, 2), embed_dim=256, num_heads=2, num_layers=2,
                                    time_budget_s=60)
    d = rep.to_json_dict()
    assert [r["cp_size"] for r in d["rows"]] == [1, 2]
    a, b = (r["max_supported_length"] for r in d["rows"])
    assert a > 0 and b >= a and "measured" in d["metadata"]["model"]


@pytest.mark.parametrize("groups", [1, 3, 8])
def test_host_streaming_fwd_bwd_matches_device_call(groups):
    # attention.hstu_attention_fwd_bwd_host: host buffers in, host results out,
    # sequence runs pipelined over copy / compute streams -- per-row results are
    # the device kernels' bitwise (sequences are independent), d_w to fp64 rounding
    from paper_2508_04711_b200 import kernels
    from paper_2508_04711_b200.attention import hstu_attention_fwd_bwd_host
    lens = [300, 0, 17, 129, 1, 64, 700, 5]
    H, d = 2, 128
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    rng = np.random.default_rng(9)
    q, k, v, g = (torch.from_numpy(rng.standard_normal((T, H * d)).astype(np.float32)).bfloat16() for _ in range(4))
    ts = torch.from_numpy(np.cumsum(rng.integers(1, 10**6, T)).astype(np.int64))
    w = oracle.normal_init_ts_weights(16, 4)
    out, dq, dk, dv, dw = hstu_attention_fwd_bwd_host(q, k, v, ts, offs, g, w, H, 16, groups=groups)
    c = lambda x: x.cuda()  # noqa: E731
    wd = torch.from_numpy(w.astype(np.float32)).cuda()
    o2 = kernels.attn_fwd(c(q), c(k), c(v), c(ts), c(ts), c(torch.from_numpy(offs)), H, wd, 16)
    q2, k2, v2, w2, _ = kernels.attn_bwd(c(q), c(k), c(v), c(ts), c(ts), c(torch.from_numpy(offs)), c(g), H, wd, 16)
    for a, b in ((out, o2), (dq, q2), (dk, k2), (dv, v2)):
        assert torch.equal(a, b.cpu())
    np.testing.assert_allclose(dw.numpy(), w2.cpu().numpy(), rtol=1e-6, atol=1e-9)


def test_host_streaming_async_back_to_back():
    # hstu_attention_fwd_bwd_host_async: three calls in flight on alternating
    # output buffers (different inputs each) give exactly the synchronous results
    from paper_2508_04711_b200.attention import hstu_attention_fwd_bwd_host, hstu_attention_fwd_bwd_host_async
    lens = [300, 17, 129, 1, 700]
    H, d = 2, 128
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    w = oracle.normal_init_ts_weights(16, 4)
    cases = []
    for seed in range(3):
        rng = np.random.default_rng(100 + seed)
        q, k, v, g = (torch.from_numpy(rng.standard_normal((T, H * d)).astype(np.float32)).bfloat16().pin_memory()
                      for _ in range(4))
        ts = torch.from_numpy(np.cumsum(rng.integers(1, 10**6, T)).astype(np.int64)).pin_memory()
        cases.append((q, k, v, ts, g))
    want = [hstu_attention_fwd_bwd_host(q, k, v, ts, offs, g, w, H, 16, groups=2) for q, k, v, ts, g in cases]
    sets = [[torch.empty((T, H * d), dtype=torch.bfloat16).pin_memory() for _ in range(4)] for _ in range(3)]
    handles = [hstu_attention_fwd_bwd_host_async(q, k, v, ts, offs, g, w, H, 16, groups=2, out=sets[i])
               for i, (q, k, v, ts, g) in enumerate(cases)]
    for hnd, ref in zip(handles, want):
        got = hnd.wait()
        for a, b in zip(got[:4], ref[:4]):
            assert torch.equal(a, b)
        np.testing.assert_allclose(got[4].numpy(), ref[4].numpy(), rtol=1e-6, atol=1e-9)


def test_attn_fwd_bwd_concurrent_equals_sequential():
    # kernels.attn_fwd_bwd (band table once, forward || backward on two streams)
    # gives exactly the results of the two calls in sequence
    from paper_2508_04711_b200 import kernels
    lens = [300, 0, 17, 129, 1, 700]
    H, d = 2, 128
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    rng = np.random.default_rng(31)
    q, k, v, g = (torch.from_numpy(rng.standard_normal((T, H * d)).astype(np.float32)).bfloat16().cuda()
                  for _ in range(4))
    ts = torch.from_numpy(np.cumsum(rng.integers(1, 10**6, T)).astype(np.int64)).cuda()
    o_ = torch.from_numpy(offs).cuda()
    w = torch.from_numpy(oracle.normal_init_ts_weights(16, 4).astype(np.float32)).cuda()
    want_o = kernels.attn_fwd(q, k, v, ts, ts, o_, H, w, 16)
    want = kernels.attn_bwd(q, k, v, ts, ts, o_, g, H, w, 16, seg_host=(offs, None, None))
    for _ in range(2):
        got = kernels.attn_fwd_bwd(q, k, v, ts, o_, g, H, w, 16, seg_host=(offs, None, None))
        torch.cuda.synchronize()
        assert torch.equal(got[0], want_o)
        for a, b in zip(got[1:4], want[:3]):
            assert torch.equal(a, b)
        np.testing.assert_allclose(got[4].cpu().numpy(), want[3].cpu().numpy(), rtol=1e-6, atol=1e-9)


def test_protocol_memory_measured():
    # all-to-all moves each rank's own share; allgather_split materialises the
    # whole group batch on every rank: its transient is larger, growing with cp
    from paper_2508_04711_b200.harness import protocol_memory_measured
    rows = protocol_memory_measured([700, 33, 1200, 5], (2, 4), embed_dim=256, num_heads=2)
    assert [r["cp_size"] for r in rows] == [2, 4]
    for r in rows:
        assert r["alltoall_peak_bytes"] > 0 and r["allgather_split_peak_bytes"] > r["alltoall_peak_bytes"]
        assert r["alltoall_resident_rows"] == r["allgather_split_resident_rows"]
    assert rows[1]["allgather_split_over_alltoall"] > rows[0]["allgather_split_over_alltoall"]
