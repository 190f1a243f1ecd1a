"""CPU checks of the drop-in boundary's host logic (no GPU calls):

* the package re-exports the reference's in-scope public names
  (jaggedcp/__init__.py:9-123);
* blockwise_partial's routing onto the kernel's segment form sees exactly the
  reference's allowed pairs (attention.py:176-183) for arbitrary seq ids /
  positions;
* ts_weights length validation (attention.py:94 indexes ts_weights by bucket);
* _map_ranks (cp_engine.py:188-206): rank-ordered results in both schedules,
  "rank r:" annotation;
* the synthetic generator's integer stream equals the reference's
  (tests/golden/synthetic.json, made by importing the reference).
"""

import json
import os

import numpy as np
import pytest
import torch

import paper_2508_04711_b200 as pkg
from paper_2508_04711_b200 import attention, cp_engine, harness, kernels

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

REFERENCE_ALL = [
    "AttentionGradients", "AttentionInputs", "BiasConfig", "BiasParams", "CollectiveError", "CommStats",
    "ExperimentConfig", "ExperimentReport", "FlopsReport", "JaggedIntSeries", "JaggedMessage", "JaggedTensor",
    "MiniChunkLayout", "PlanEntry", "QKVBatch", "RankContext", "RankGroup", "ShardPlan", "SweepReport",
    "all_gather_jagged", "all_to_all_jagged", "blockwise_partial", "bucketize", "build_shard_plan",
    "chunk_assignment", "compute_bias", "flops_per_rank", "gen_synthetic_batch", "hstu_attention_backward",
    "hstu_attention_reference", "inverse_reorder", "lengths", "make_minichunks", "new_int_series", "new_jagged",
    "redistribute_allgather_split", "redistribute_alltoall", "reorder_balanced", "restore_outputs",
    "ring_hstu_attention", "ring_send_recv", "run_experiment", "run_pipeline", "silu", "sweep_max_tokens",
]
# out of scope: record serialisation, verification grid, fixture bundles
OUT_OF_SCOPE = {"jagged_from_record", "jagged_to_record", "verify_grid", "VerifyReport", "fixture_bundle"}


def test_package_exports_reference_names():
    for name in REFERENCE_ALL:
        assert hasattr(pkg, name), name
        assert name in pkg.__all__, name
    assert not (OUT_OF_SCOPE & set(pkg.__all__))


def _allowed(qs, qp, ks, kp):
    return (qs[:, None] == ks[None, :]) & (kp[None, :] <= qp[:, None])


def _routed(qs, qp, ks, kp):
    q_perm, k_perm, offs, pos0, kvs, kvl = attention._blockwise_segments(qs, qp, ks, kp)
    got = np.zeros((qs.size, ks.size), dtype=bool)
    assert offs[0] == 0 and offs[-1] == qs.size and np.all(np.diff(offs) > 0)
    assert sorted(q_perm.tolist()) == list(range(qs.size)) and sorted(k_perm.tolist()) == list(range(ks.size))
    for s in range(offs.size - 1):
        for i in range(offs[s], offs[s + 1]):
            qpos = pos0[s] + (i - offs[s])
            for j in range(kvl[s]):
                if j <= qpos:
                    got[q_perm[i], k_perm[kvs[s] + j]] = True
    return got


@pytest.mark.parametrize("seed", range(12))
def test_blockwise_routing_matches_reference_mask(seed):
    rng = np.random.default_rng(seed)
    nq, nk = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    nseq, npos = int(rng.integers(1, 4)), int(rng.integers(1, 25))
    qs, ks = rng.integers(0, nseq, nq), rng.integers(0, nseq, nk)
    qp, kp = rng.integers(0, npos, nq), rng.integers(0, npos, nk)
    np.testing.assert_array_equal(_routed(qs, qp, ks, kp), _allowed(qs, qp, ks, kp))


def test_blockwise_routing_golden_and_runs():
    d = np.load(os.path.join(GOLDEN, "blockwise_cases.npz"))
    qs, qp, ks, kp = d["b0/qs"], d["b0/qp"], d["b0/ks"], d["b0/kp"]
    np.testing.assert_array_equal(_routed(qs, qp, ks, kp), _allowed(qs, qp, ks, kp))
    # CP ring shape: resident chunk rows x one visiting chunk (consecutive runs) -> few segments
    qs = np.repeat([0, 1], [50, 30])
    qp = np.concatenate([np.arange(100, 150), np.arange(0, 30)])
    ks = np.repeat([0, 1], [40, 20])
    kp = np.concatenate([np.arange(60, 100), np.arange(10, 30)])
    np.testing.assert_array_equal(_routed(qs, qp, ks, kp), _allowed(qs, qp, ks, kp))
    assert attention._blockwise_segments(qs, qp, ks, kp)[2].size - 1 <= 3


def test_ts_weights_length_validated():
    with pytest.raises(ValueError, match="num_buckets"):
        kernels._check_weights(torch.zeros(8), 16)
    with pytest.raises(ValueError, match="num_buckets"):
        kernels._check_weights(torch.zeros(2, 16), 16)
    kernels._check_weights(torch.zeros(16), 16)
    assert kernels.padded_head_dim(8) == 64 and kernels.padded_head_dim(96) == 128
    with pytest.raises(NotImplementedError):
        kernels.padded_head_dim(256)
    x = torch.arange(2 * 3 * 8, dtype=torch.float32).view(2, 24)
    assert torch.equal(kernels._unpad_heads(kernels._pad_heads(x, 3, 8, 64), 3, 8, 64), x)


@pytest.mark.parametrize("sched", ["sequential", "threaded"])
def test_map_ranks_order_and_annotation(sched):
    assert cp_engine._map_ranks(lambda r: r * r, 5, sched) == [0, 1, 4, 9, 16]

    def bad(r):
        if r == 2:
            raise ValueError("boom")
        return r

    with pytest.raises(RuntimeError, match="rank 2: boom"):
        cp_engine._map_ranks(bad, 4, sched)
    with pytest.raises(ValueError, match="scheduling"):
        cp_engine._map_ranks(bad, 2, "parallel")


def test_generator_matches_reference_integer_stream():
    with open(os.path.join(GOLDEN, "synthetic.json")) as f:
        cases = json.load(f)
    for c in cases:
        kw = dict(c["cfg"])
        if kw["dtype"] == "f64":
            kw["dtype"] = "bf16"  # this repo's tag draws the reference's f64 stream
        h = harness.gen_synthetic_host(harness.ExperimentConfig(**kw), c["rank"])
        assert h["offsets"].tolist() == c["offsets"], c["cfg"]
        assert h["ts"].tolist() == c["ts"], c["cfg"]
        assert abs(float(np.asarray(h["q"], np.float64).sum()) - c["q_sum"]) <= 1e-9 * max(1.0, abs(c["q_sum"]))


@pytest.mark.parametrize("G", [1, 2, 3, 8, 40])
def test_host_streaming_cut_points(G):
    # the host-streaming call's runs: whole sequences, every sequence in exactly
    # one run, G clamped to the sequence count, ~T/G tokens per run
    from paper_2508_04711_b200.attention import _stream_cuts
    rng = np.random.default_rng(G)
    lens = rng.integers(0, 1025, 32)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    g = max(1, min(G, lens.size))
    cuts = _stream_cuts(offs, g)
    assert cuts[0] == 0 and cuts[-1] == lens.size and len(cuts) == g + 1
    assert all(b > a for a, b in zip(cuts, cuts[1:]))  # no empty run of sequences
    sizes = [int(offs[b] - offs[a]) for a, b in zip(cuts, cuts[1:])]
    assert sum(sizes) == int(offs[-1])
    if g > 1:
        assert max(sizes) <= int(offs[-1]) / g + int(lens.max())  # within one sequence of the even share


def test_bench_reference_arm_under_torchrun():
    # the driver launches --impl reference like the GPU arm (torchrun for N > 1):
    # rank 0 alone runs the reference's CPU path and prints the one JSON line
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", f"--master-port={port}", os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
    assert j["e2e"]["value"] == j["value"] and j["cpu_baseline"]["kind"] in ("reference", "port")
