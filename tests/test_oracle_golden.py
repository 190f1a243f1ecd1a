"""Pin the CPU oracle (oracle/) to the reference.

The golden fixtures under tests/golden/ were produced by importing the
unmodified reference package (tests/golden/make_golden.py).  The literal
known-answer values below are the ones the reference's own test-suite pins
(test_attention.py, test_jagged.py, test_cp_engine.py).
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import attention as oa
from oracle import harness as oh
from conftest import GOLDEN, load_npz_cases


# ---- known-answer tests from the reference suite -----------------------------

def test_silu_known_answers():  # test_attention.py:24-36
    assert oa.silu(0.0) == 0.0
    assert float(oa.silu(1.0)) == pytest.approx(0.7310585786300049, abs=1e-15)
    assert float(oa.silu(-20.0)) == pytest.approx(-4.122307244877116e-08, rel=1e-9)
    assert float(oa.silu(-800.0)) == 0.0


def test_bucketize_known_answers():  # test_attention.py:46-67
    assert oa.bucketize(0, 16) == 0
    assert oa.bucketize(10, 16) == 2
    assert oa.bucketize(10**9, 16) == 15
    assert oa.bucketize(-12345, 16) == 0


def test_compute_bias_known_answer():  # test_attention.py:78-84
    w = np.zeros(16)
    w[2] = 0.5
    assert oa.compute_bias([100], [90], w, 16).tolist() == [[0.5]]


def test_length_one_closed_form():  # test_attention.py:107-114
    d = 4
    w = np.zeros(4)
    w[0] = 0.125
    out = oa.hstu_forward(np.full((1, d), 0.5), np.full((1, d), 0.25), np.full((1, d), 2.0),
                          np.array([7]), [0, 1], w, 4)
    s = (0.5 * 0.25 * d + 0.125) / math.sqrt(d)
    assert np.allclose(out, float(oa.silu(s)) * 2.0, atol=1e-15)


def test_minichunk_known_answers():  # test_jagged.py:66-105
    assert oracle.make_minichunks([8], 2)[2][0] == (2, 2, 2, 2)
    assert oracle.make_minichunks([10], 2)[2][0] == (3, 3, 2, 2)
    assert oracle.make_minichunks([3], 4)[2][0] == (1, 1, 1, 0, 0, 0, 0, 0)
    assert oracle.chunk_assignment(4) == {0: (0, 7), 1: (1, 6), 2: (2, 5), 3: (3, 4)}


def test_flops_known_answers():  # test_cp_engine.py:246-265
    assert oracle.flops_per_rank(oracle.build_shard_plan([[8], []], 2, "balanced_minichunk"))[0] == (18, 18)
    pr, tot, ratio = oracle.flops_per_rank(oracle.build_shard_plan([[8], []], 2, "naive_contiguous"))
    assert pr == (10, 26) and ratio == pytest.approx(26 / 18, abs=1e-12)
    _, _, r8 = oracle.flops_per_rank(oracle.build_shard_plan([[4096]] + [[]] * 7, 8, "naive_contiguous"))
    assert abs(r8 - 1.875) / 1.875 < 0.02


# ---- golden fixtures produced by the reference itself ----------------------

@pytest.mark.parametrize("name", sorted(load_npz_cases("attention_cases.npz")))
def test_attention_matches_reference_fixture(name):
    c = load_npz_cases("attention_cases.npz")[name]
    H, nb = (int(x) for x in c["meta"])
    o = oa.hstu_forward(c["q"], c["k"], c["v"], c["ts"], c["offsets"], c["w"], nb, H)
    dq, dk, dv, dw, _ = oa.hstu_backward(c["q"], c["k"], c["v"], c["ts"], c["offsets"], c["g"], c["w"], nb, H)
    tol = 1e-12 if c["q"].dtype == np.float64 else 2e-4
    for got, want in ((o, c["o"]), (dq, c["dq"]), (dk, c["dk"]), (dv, c["dv"])):
        assert oh.output_errors([got], [want])[1] <= tol
    assert np.allclose(dw, c["dw"], rtol=1e-9, atol=1e-9 if c["q"].dtype == np.float64 else 1e-5)


def test_blockwise_matches_reference_fixture():
    c = load_npz_cases("blockwise_cases.npz")["b0"]
    got = oa.blockwise_partial(c["q"], c["qs"], c["qp"], c["tq"], c["k"], c["ks"], c["kp"], c["tk"], c["v"], c["w"], 16)
    assert np.abs(got - c["out"]).max() < 1e-12


def test_buckets_match_reference_fixture():
    d = np.load(os.path.join(GOLDEN, "buckets.npz"))
    for key in d.files:
        if key.startswith("nb"):
            assert np.array_equal(oa.bucketize_array(d["deltas"], int(key[2:])), d[key]), key


def test_plans_match_reference_fixture():
    rec = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for p in rec["plans"]:
        plan = oracle.build_shard_plan(p["lengths_per_rank"], p["cp"], p["mode"])
        assert list(plan["seq_owner"]) == p["seq_owner"]
        assert list(plan["chunk_owner"]) == p["chunk_owner"]
        assert [list(x) for x in plan["layout"][2]] == p["chunk_lengths"]
        assert [[list(e) for e in ents] for ents in plan["rank_entries"]] == p["rank_entries"]
        pr, tot, ratio = oracle.flops_per_rank(plan)
        assert list(pr) == p["flops_per_rank"] and tot == p["flops_total"]
        assert ratio == pytest.approx(p["max_mean_ratio"], rel=1e-15)
    for r in rec["reorders"]:
        offs = np.concatenate([[0], np.cumsum(r["lengths"])])
        layout = oracle.make_minichunks(r["lengths"], r["cp"])
        perm, _ = oracle.rank_major_row_order(offs, layout)
        assert perm.tolist() == r["perm"]
        assert [list(x) for x in oracle.rank_row_ranges(layout)] == r["rank_row_ranges"]


def test_synthetic_generator_matches_reference():
    rec = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for s in rec["synthetic"]:
        b = oh.gen_synthetic_batch(s["seed"], s["rank"], s["batch_size"], 8, np.float32, s["dist"], 1,
                                   s["max_len"], float(np.log(1024)), 1.0, max(s["max_len"], 8192))
        assert np.diff(b["offsets"]).tolist() == s["lengths"]
        assert int(b["ts"].sum()) == s["ts_sum"] and int(b["ts"][0]) == s["ts_first"]
        assert float(b["q"][0, 0]) == s["q00"] and float(b["v"][-1, -1]) == s["v_last"]


def test_golden_experiment_plan_fields():
    # reference tests/golden/bench_cp2_seed23.json: resident tokens [27, 25], flops [235, 242]
    rec = json.load(open(os.path.join(GOLDEN, "plans.json")))["experiment"]
    assert rec["resident_tokens_per_rank"] == [27, 25]
    assert rec["flops"]["per_rank"] == [235, 242]
    b = [oh.gen_synthetic_batch(23, r, 2, 8, np.float64, "uniform", 0, 24, 3.0, 0.8, 32) for r in range(2)]
    plan = oracle.build_shard_plan([np.diff(x["offsets"]).tolist() for x in b], 2, "balanced_minichunk")
    assert [sum(e - s for (_, _, s, e) in ents) for ents in plan["rank_entries"]] == [27, 25]
    assert list(oracle.flops_per_rank(plan)[0]) == [235, 242]


def test_cp_sim_matches_reference_pipeline():
    cases = load_npz_cases("cp_cases.npz")
    for tag, c in cases.items():
        cp = int(tag.split("_")[0][2:])
        mode = "balanced_minichunk" if "balanced" in tag else "naive_contiguous"
        seed = int(tag.split("_")[-1])
        batches = [oh.gen_synthetic_batch(seed, r, 3, 16, np.float64, "uniform", 0, 40, 3.0, 0.8, 64) for r in range(cp)]
        outs, _ = oracle.cp_forward_sim(batches, cp, mode, c["w"], 16, 1)
        for r in range(cp):
            assert np.abs(outs[r] - c[f"out{r}"]).max() < 1e-10
