"""Freeze reference outputs into small golden fixtures.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference package ``jaggedcp`` from
``/root/reference/pkg/src`` and records, for seeded inputs, the values the
oracle (``oracle/``) and the CUDA path are checked against:

* ``attention_cases.npz``  - single-device forward/backward
  (``hstu_attention_reference`` attention.py:125, ``hstu_attention_backward``
  attention.py:187) on small jagged batches, f64 and f32, including empty
  and length-1 sequences, plus a bf16-rounded 2-head d=64 case (config C1
  shape, lengths <= 64) run per head.
* ``blockwise_cases.npz``  - ``blockwise_partial`` (attention.py:151).
* ``buckets.npz``          - ``bucketize_array`` (attention.py:83) around every
  threshold e^k - 1 for k <= 45, plus random/negative/huge deltas, for several
  ``num_buckets``.
* ``plans.json``           - ``build_shard_plan``/``flops_per_rank``
  (cp_engine.py:105,528), ``reorder_balanced`` permutations and
  ``rank_row_ranges`` (jagged.py:221,232), synthetic-batch checksums
  (harness.py:123) and the integer fields of ``run_experiment`` for the
  reference's own golden config (tests/golden/bench_cp2_seed23.json).
* ``cp_cases.npz``         - ``run_pipeline`` outputs (cp_engine.py:563).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import jaggedcp  # noqa: E402
    from jaggedcp import harness, jagged  # noqa: E402
    return jaggedcp, harness, jagged


def _bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def attention_cases(jc):
    out = {}
    cases = [
        # name, lengths, d, heads, dtype, nb, seed
        ("f64_mixed", [5, 0, 17, 1, 32], 8, 1, np.float64, 16, 1),
        ("f64_single1", [1], 4, 1, np.float64, 16, 2),
        ("f32_mixed", [33, 2, 0, 48], 16, 1, np.float32, 16, 3),
        ("f64_nb8", [40, 9], 8, 1, np.float64, 8, 4),
        ("f32_c1_bf16", [64, 17, 50, 31], 128, 2, np.float32, 16, 7),
        ("f32_d64_bf16_long", [200, 129, 128, 1], 64, 1, np.float32, 16, 9),
    ]
    for name, lens, D, H, dt, nb, seed in cases:
        rng = np.random.default_rng(seed)
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        T = int(offs[-1])
        q, k, v, g = (rng.standard_normal((T, D)).astype(dt) for _ in range(4))
        if "bf16" in name:
            q, k, v, g = (_bf16_round(a).astype(dt) for a in (q, k, v, g))
        ts = np.zeros(T, dtype=np.int64)
        for b, L in enumerate(lens):
            lo = int(offs[b])
            ts[lo:lo + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, 1_000_001, size=L))
        w = jc.BiasParams.normal_init(jc.BiasConfig(nb), seed + 0x5EED).ts_weights
        d = D // H
        o = np.zeros_like(v)
        dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
        dw = np.zeros(nb)
        for h in range(H):
            cs = slice(h * d, (h + 1) * d)
            mk = lambda a: jc.new_jagged(np.ascontiguousarray(a[:, cs]), offs, max(lens))  # noqa: E731
            inp = jc.AttentionInputs(mk(q), mk(k), mk(v), jc.new_int_series(ts, offs),
                                     jc.BiasParams(w), jc.BiasConfig(nb))
            o[:, cs] = jc.hstu_attention_reference(inp).values
            gr = jc.hstu_attention_backward(inp, mk(g))
            dq[:, cs], dk[:, cs], dv[:, cs] = gr.dq.values, gr.dk.values, gr.dv.values
            dw += gr.d_ts_weights
        for key, val in dict(q=q, k=k, v=v, g=g, ts=ts, offsets=offs, w=w, o=o, dq=dq, dk=dk, dv=dv,
                             dw=dw, meta=np.array([H, nb], dtype=np.int64)).items():
            out[f"{name}/{key}"] = val
    np.savez_compressed(os.path.join(HERE, "attention_cases.npz"), **out)


def blockwise_cases(jc):
    rng = np.random.default_rng(11)
    out = {}
    nq, nk, d = 13, 9, 8
    q, k, v = (rng.standard_normal((n, d)) for n in (nq, nk, nk))
    qs = rng.integers(0, 3, nq)
    qp = rng.integers(0, 20, nq)
    ks = rng.integers(0, 3, nk)
    kp = rng.integers(0, 20, nk)
    tq = rng.integers(0, 10**7, nq)
    tk = rng.integers(0, 10**7, nk)
    w = jc.BiasParams.normal_init(jc.BiasConfig(16), 5).ts_weights
    res = jc.blockwise_partial(q, qs, qp, tq, k, ks, kp, tk, v, jc.BiasParams(w), jc.BiasConfig(16))
    for key, val in dict(q=q, k=k, v=v, qs=qs, qp=qp, ks=ks, kp=kp, tq=tq, tk=tk, w=w, out=res).items():
        out[f"b0/{key}"] = val
    np.savez_compressed(os.path.join(HERE, "blockwise_cases.npz"), **out)


def bucket_cases(jc):
    from jaggedcp.attention import bucketize_array
    deltas = [0, 1, 2, 3, -1, -12345, 10, 10**9, 2**62, -(2**62), 2**63 - 1, -(2**63)]
    for kk in range(1, 46):
        t = int(np.ceil(np.exp(kk) - 1.0)) if kk < 43 else int(min(np.exp(kk), 2**63 - 2048))
        for dd in range(-3, 4):
            x = t + dd
            if -(2**63) <= x < 2**63:
                deltas.append(x)
    rng = np.random.default_rng(3)
    deltas += [int(x) for x in rng.integers(-10**6, 10**7, 4000)]
    deltas += [int(x) for x in rng.integers(0, 2**62, 500)]
    deltas = np.asarray(deltas, dtype=np.int64)
    out = {"deltas": deltas}
    for nb in (1, 2, 8, 16, 33, 40, 64):
        out[f"nb{nb}"] = bucketize_array(deltas, jc.BiasConfig(nb))
    np.savez_compressed(os.path.join(HERE, "buckets.npz"), **out)


def plans(jc, harness, jagged):
    rec = {"plans": [], "reorders": [], "synthetic": [], "experiment": {}}
    cases = [
        ([[16], [], [], []], 4, "balanced_minichunk"),
        ([[8], []], 2, "naive_contiguous"),
        ([[5, 3]], 1, "balanced_minichunk"),
        ([[7, 0], [13, 2]], 2, "balanced_minichunk"),
        ([[12], [], [9]], 3, "balanced_minichunk"),
        ([[1000, 3, 0, 77], [5, 4096], [17], [2, 2]], 4, "balanced_minichunk"),
        ([[1000, 3, 0, 77], [5, 4096], [17], [2, 2]], 4, "naive_contiguous"),
        ([[33, 1, 8191, 0], [640], [1, 1], [9], [100, 101], [3], [7], [8192]], 8, "balanced_minichunk"),
        ([[33, 1, 8191, 0], [640], [1, 1], [9], [100, 101], [3], [7], [8192]], 8, "naive_contiguous"),
    ]
    for lpr, cp, mode in cases:
        plan = jc.build_shard_plan(lpr, cp, mode)
        fl = jc.flops_per_rank(plan)
        rec["plans"].append({
            "lengths_per_rank": lpr, "cp": cp, "mode": mode,
            "seq_owner": list(plan.seq_owner), "chunk_owner": list(plan.chunk_owner),
            "chunk_lengths": [list(x) for x in plan.layout.chunk_lengths],
            "rank_entries": [[[e.seq_id, e.chunk_id, e.start, e.end] for e in ents] for ents in plan.rank_entries],
            "flops_per_rank": list(fl.per_rank), "flops_total": fl.total, "max_mean_ratio": fl.max_mean_ratio,
        })
    for lens, cp in (([8], 2), ([4, 4], 2), ([13, 0, 7, 100], 3), ([1000, 1, 2, 3, 513], 4), ([5, 3], 1)):
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        jt = jc.new_jagged(np.zeros((int(offs[-1]), 1)), offs, max(lens))
        layout = jc.make_minichunks(lens, cp)
        _, perm = jc.reorder_balanced(jt, layout)
        rec["reorders"].append({"lengths": lens, "cp": cp, "perm": [int(x) for x in perm],
                                "rank_row_ranges": [list(x) for x in jagged.rank_row_ranges(layout)]})
    for seed, rank, bs, dist, mx in ((7, 0, 4, "uniform", 256), (7, 0, 32, "uniform", 1024),
                                     (7, 1, 16, "uniform", 4096), (7, 3, 4, "lognormal", 8192)):
        cfg = harness.ExperimentConfig(cp_size=max(rank + 1, 1), batch_size=bs, length_dist=dist, min_len=1,
                                       max_len=mx, max_length=max(mx, 8192), lognorm_mu=float(np.log(1024)),
                                       lognorm_sigma=1.0, embed_dim=8, dtype="f32", seed=seed)
        b = harness.gen_synthetic_batch(cfg, rank)
        rec["synthetic"].append({
            "seed": seed, "rank": rank, "batch_size": bs, "dist": dist, "max_len": mx,
            "lengths": [int(x) for x in np.diff(b.q.offsets)],
            "ts_sum": int(b.ts.values.sum()), "ts_first": int(b.ts.values[0]),
            "q00": float(b.q.values[0, 0]), "v_last": float(b.v.values[-1, -1]),
        })
    cfg = harness.ExperimentConfig(cp_size=2, batch_size=2, min_len=0, max_len=24, max_length=32, embed_dim=8, seed=23)
    rep = harness.run_experiment(cfg).to_json_dict()
    rec["experiment"] = {
        "config": rep["config"],
        "resident_tokens_per_rank": rep["resident_tokens_per_rank"],
        "flops": rep["flops"],
    }
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)


def cp_cases(jc, harness):
    out = {}
    for cp, mode, seed in ((2, "balanced_minichunk", 5), (4, "naive_contiguous", 6), (4, "balanced_minichunk", 8)):
        cfg = harness.ExperimentConfig(cp_size=cp, batch_size=3, min_len=0, max_len=40, max_length=64,
                                       embed_dim=16, dtype="f64", seed=seed, balance_mode=mode)
        batches = [harness.gen_synthetic_batch(cfg, r) for r in range(cp)]
        params, bcfg = harness.bias_for_config(cfg)
        res = jc.run_pipeline(batches, cp, "alltoall", mode, params, bcfg)
        tag = f"cp{cp}_{mode}_{seed}"
        out[f"{tag}/w"] = params.ts_weights
        for r in range(cp):
            out[f"{tag}/out{r}"] = res.outputs[r].values
            out[f"{tag}/offsets{r}"] = res.outputs[r].offsets
    np.savez_compressed(os.path.join(HERE, "cp_cases.npz"), **out)


def main():
    jc, harness, jagged = _ref()
    attention_cases(jc)
    blockwise_cases(jc)
    bucket_cases(jc)
    plans(jc, harness, jagged)
    cp_cases(jc, harness)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
