"""Numpy restatement of the reference CP plan and pipeline (TEST ORACLE).

Follows ``/root/reference/pkg/src/jaggedcp/cp_engine.py``:

* ``build_shard_plan`` -> cp_engine.py:105-147.  Returns a dict with
  ``seq_lengths``, ``seq_owner``, ``chunk_owner``, ``layout`` and
  ``rank_entries`` = per rank a list of ``(seq_id, chunk_id, start, end)``
  ordered by sequence then chunk (cp_engine.py:131-137).
* ``flops_per_rank``   -> cp_engine.py:528-548 (exact causal-pair counts).
* ``cp_forward_sim``   -> run_pipeline (cp_engine.py:563-598) restated as
  plan -> route rows to owners -> per-rank blockwise sums -> restore.
"""

from __future__ import annotations

import numpy as np

from .attention import hstu_fwd_seq, silu, compute_bias
from .jagged import chunk_owner_map, make_contiguous_chunks, make_minichunks

BALANCE_MODES = ("balanced_minichunk", "naive_contiguous")


def build_shard_plan(lengths_per_rank, cp_size: int, balance_mode: str) -> dict:
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    if balance_mode not in BALANCE_MODES:
        raise ValueError(f"unknown balance_mode {balance_mode!r}")
    if len(lengths_per_rank) != cp_size:
        raise ValueError(f"expected {cp_size} per-rank length lists, got {len(lengths_per_rank)}")
    seq_lengths, seq_owner = [], []
    for rank, ls in enumerate(lengths_per_rank):
        seq_lengths.extend(int(x) for x in ls)
        seq_owner.extend([rank] * len(ls))
    layout = (make_minichunks if balance_mode == "balanced_minichunk" else make_contiguous_chunks)(seq_lengths, cp_size)
    owners = chunk_owner_map(layout)
    ranges = layout[3]
    rank_entries = []
    for r in range(cp_size):
        rank_entries.append([
            (b, c, ranges[b][c][0], ranges[b][c][1])
            for b in range(len(seq_lengths))
            for c in range(layout[1])
            if owners[c] == r
        ])
    return {
        "cp_size": cp_size,
        "balance_mode": balance_mode,
        "seq_lengths": tuple(seq_lengths),
        "seq_owner": tuple(seq_owner),
        "layout": layout,
        "chunk_owner": owners,
        "rank_entries": rank_entries,
    }


def flops_per_rank(plan: dict):
    def tri(n: int) -> int:
        return n * (n + 1) // 2

    per_rank = tuple(sum(tri(e) - tri(s) for (_, _, s, e) in ents) for ents in plan["rank_entries"])
    total = sum(tri(L) for L in plan["seq_lengths"])
    ratio = 1.0 if total == 0 else max(per_rank) / (total / plan["cp_size"])
    return per_rank, total, ratio


def cp_forward_sim(batches, cp_size, balance_mode, ts_weights, num_buckets=16, num_heads=1):
    """batches: list over ranks of dicts {q,k,v,ts,offsets}.  Returns the
    per-rank restored outputs (same row order as each rank's input)."""
    plan = build_shard_plan([np.diff(b["offsets"]).tolist() for b in batches], cp_size, balance_mode)
    # combined (group) view, sequences in rank order (harness.concat_batches)
    q = np.concatenate([b["q"] for b in batches])
    k = np.concatenate([b["k"] for b in batches])
    v = np.concatenate([b["v"] for b in batches])
    ts = np.concatenate([b["ts"] for b in batches])
    goff = np.concatenate([[0], np.cumsum(plan["seq_lengths"])]).astype(np.int64)
    D = q.shape[1]
    d = D // num_heads
    out = np.zeros_like(v)
    # every rank: resident q chunks x all visiting kv chunks of the same
    # sequence (ring sum == full causal prefix), summed in chunk order
    for r in range(cp_size):
        for (b, c, s, e) in plan["rank_entries"][r]:
            if e == s:
                continue
            base = int(goff[b])
            for h in range(num_heads):
                cs = slice(h * d, (h + 1) * d)
                qb = q[base + s:base + e, cs]
                acc = np.zeros((e - s, d), dtype=q.dtype)
                for (c2_start, c2_end) in plan["layout"][3][b]:
                    if c2_end == c2_start or c2_start > e - 1:
                        continue
                    kb = k[base + c2_start:base + c2_end, cs]
                    vb = v[base + c2_start:base + c2_end, cs]
                    scale = q.dtype.type(np.sqrt(d))
                    bias = compute_bias(ts[base + s:base + e], ts[base + c2_start:base + c2_end],
                                        ts_weights, num_buckets).astype(q.dtype)
                    sc = silu((qb @ kb.T + bias) / scale)
                    allowed = np.arange(c2_start, c2_end)[None, :] <= np.arange(s, e)[:, None]
                    acc += np.where(allowed, sc, q.dtype.type(0)) @ vb
                out[base + s:base + e, cs] = acc
    # restore: split the group rows back per contributing rank
    res, row = [], 0
    for bt in batches:
        n = bt["q"].shape[0]
        res.append(out[row:row + n])
        row += n
    return res, plan


__all__ = ["build_shard_plan", "flops_per_rank", "cp_forward_sim", "hstu_fwd_seq"]
