"""Jagged context parallelism (mirror of ``jaggedcp/cp_engine.py``).

Plan types and the exact integer plan (cp_engine.py:48-147, 528-548) come
from the C ABI; the data path (redistribution, KV exchange, attention,
restore) runs on the GPU -- see ``cp_layer.py`` for the SPMD (one process per
GPU, torch.distributed/NCCL) layer and the global-view functions below for
the reference's single-process signatures.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check
from .jagged import JaggedIntSeries, JaggedTensor, MiniChunkLayout, _plan_arrays, lengths

BALANCE_MODES = ("balanced_minichunk", "naive_contiguous")


def _mode(balance_mode: str) -> int:
    if balance_mode not in BALANCE_MODES:
        raise ValueError(f"unknown balance_mode {balance_mode!r}")
    return 0 if balance_mode == "balanced_minichunk" else 1


@dataclass(frozen=True)
class QKVBatch:
    """cp_engine.py:48-67: one rank's local attention inputs."""

    q: JaggedTensor
    k: JaggedTensor
    v: JaggedTensor
    ts: JaggedIntSeries

    def __post_init__(self) -> None:
        for name, t in (("k", self.k), ("v", self.v), ("ts", self.ts)):
            if not np.array_equal(self.q.host_offsets, t.host_offsets):
                raise ValueError(f"offsets of q and {name} differ")

    @property
    def num_sequences(self) -> int:
        return self.q.num_sequences

    def payload_nbytes(self) -> int:
        return sum(t.values.numel() * t.values.element_size() for t in (self.q, self.k, self.v, self.ts))


@dataclass(frozen=True)
class PlanEntry:
    """cp_engine.py:70-79."""

    seq_id: int
    chunk_id: int
    start: int
    end: int

    @property
    def count(self) -> int:
        return self.end - self.start


@dataclass(frozen=True)
class ShardPlan:
    """cp_engine.py:82-102."""

    cp_size: int
    balance_mode: str
    seq_lengths: tuple
    seq_owner: tuple
    layout: MiniChunkLayout
    chunk_owner: tuple
    rank_entries: tuple

    @property
    def num_sequences(self) -> int:
        return len(self.seq_lengths)

    def group_offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.seq_lengths)]).astype(np.int64)

    def rank_token_counts(self) -> tuple:
        return tuple(sum(e.count for e in entries) for entries in self.rank_entries)


def build_shard_plan(lengths_per_rank: Sequence[Sequence[int]], cp_size: int, balance_mode: str) -> ShardPlan:
    """cp_engine.py:105-147 (integers from jh_plan_build, bit-exact)."""
    if cp_size < 1:
        raise ValueError("cp_size must be >= 1")
    mode = _mode(balance_mode)
    if len(lengths_per_rank) != cp_size:
        raise ValueError(f"expected {cp_size} per-rank length lists, got {len(lengths_per_rank)}")
    seq_lengths, seq_owner = [], []
    for rank, ls in enumerate(lengths_per_rank):
        seq_lengths.extend(int(x) for x in ls)
        seq_owner.extend([rank] * len(ls))
    cl, cs, co = _plan_arrays(seq_lengths, cp_size, mode)
    C = len(co)
    layout = MiniChunkLayout(
        cp_size, C, tuple(tuple(int(x) for x in row) for row in cl),
        tuple(tuple((int(cs[b, c]), int(cs[b, c] + cl[b, c])) for c in range(C)) for b in range(len(seq_lengths))))
    owners = tuple(int(x) for x in co)
    rank_entries = tuple(
        tuple(PlanEntry(b, c, *layout.chunk_ranges[b][c]) for b in range(len(seq_lengths)) for c in range(C)
              if owners[c] == r)
        for r in range(cp_size))
    return ShardPlan(cp_size, balance_mode, tuple(seq_lengths), tuple(seq_owner), layout, owners, rank_entries)


@dataclass(frozen=True)
class FlopsReport:
    """cp_engine.py:172-185."""

    per_rank: tuple
    total: int
    max_mean_ratio: float

    def to_json_dict(self) -> dict:
        return {"per_rank": list(self.per_rank), "total": self.total, "max_mean_ratio": self.max_mean_ratio}


def flops_per_rank(plan: ShardPlan, seq_lengths: Sequence[int] | None = None) -> FlopsReport:
    """cp_engine.py:528-548 (exact causal pair counts, jh_flops_per_rank)."""
    if seq_lengths is not None and tuple(int(x) for x in seq_lengths) != plan.seq_lengths:
        raise ValueError("seq_lengths do not match the plan")
    lens = np.ascontiguousarray(np.asarray(plan.seq_lengths, dtype=np.int64))
    pr = np.zeros(plan.cp_size, dtype=np.int64)
    tot = ctypes.c_int64()
    P64 = ctypes.POINTER(ctypes.c_int64)
    check(_lib.lib().jh_flops_per_rank(lens.ctypes.data_as(P64) if lens.size else None, lens.size, plan.cp_size,
                                       _mode(plan.balance_mode), pr.ctypes.data_as(P64), ctypes.byref(tot)),
          "flops_per_rank")
    total = int(tot.value)
    ratio = 1.0 if total == 0 else max(int(x) for x in pr) / (total / plan.cp_size)
    return FlopsReport(tuple(int(x) for x in pr), total, ratio)


def plan_from_batches(batches: Sequence[QKVBatch], cp_size: int, balance_mode: str) -> ShardPlan:
    return build_shard_plan([lengths(b.q).tolist() for b in batches], cp_size, balance_mode)


# ----------------------------------------------------------------------------
# Global-view (single-process) pipeline with the reference's signatures.
# All ranks' data sit on one device; routing is device-side row gathers, the
# attention is the fused sm_100a kernel over per-chunk segments.
# ----------------------------------------------------------------------------

import torch  # noqa: E402

from . import kernels  # noqa: E402
from .comm import (CommStats, JaggedMessage, MemoryMeter, RankGroup, all_to_all_jagged,  # noqa: E402
                   gather_traffic)
from .jagged import JaggedTensor  # noqa: E402

SCHEDULINGS = ("sequential", "threaded")


@dataclass
class RankContext:
    """cp_engine.py:150-169: one rank's resident rows (plan order) + provenance."""

    rank: int
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    ts: torch.Tensor
    seq_ids: np.ndarray
    positions: np.ndarray
    chunk_ids: np.ndarray
    entries: tuple

    @property
    def num_rows(self) -> int:
        return self.q.shape[0]

    def payload_nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in (self.q, self.k, self.v, self.ts))


def _check_sched(scheduling: str) -> None:
    if scheduling not in SCHEDULINGS:
        raise ValueError(f"unknown scheduling {scheduling!r}")


def _map_ranks(fn, cp_size: int, scheduling: str, devices=None) -> list:
    """cp_engine.py:188-206: run a per-rank function sequentially or on a
    thread pool (kernel launches are thread-safe; every rank's work is
    stream-ordered on the current stream of ITS device -- ``devices[r]`` in
    the single-process multi-device mode); results in rank order, failures
    re-raised as RuntimeError("rank r: ...")."""

    def run(r: int):
        try:
            dev = None if devices is None else devices[r]
            if dev is not None and dev.type == "cuda":
                with torch.cuda.device(dev):
                    return fn(r)
            return fn(r)
        except Exception as exc:  # annotate with the failing rank
            raise RuntimeError(f"rank {r}: {exc}") from exc

    if scheduling == "threaded" and cp_size > 1:
        from concurrent.futures import ThreadPoolExecutor
        cuda = torch.cuda.is_available()
        streams = [torch.cuda.current_stream(None if devices is None else devices[r]) if cuda else None
                   for r in range(cp_size)]

        def run_on_stream(r: int):
            if streams[r] is None:
                return run(r)
            with torch.cuda.stream(streams[r]):
                return run(r)

        with ThreadPoolExecutor(max_workers=cp_size) as pool:
            futures = [pool.submit(run_on_stream, r) for r in range(cp_size)]
            return [f.result() for f in futures]
    _check_sched(scheduling)
    return [run(r) for r in range(cp_size)]


def _entries_meta(entries):
    """cp_engine.py:209-213."""
    if not entries:
        z = np.zeros(0, np.int64)
        return z, z.copy(), z.copy()
    seq = np.concatenate([np.full(e.count, e.seq_id, np.int64) for e in entries])
    pos = np.concatenate([np.arange(e.start, e.end, dtype=np.int64) for e in entries])
    chk = np.concatenate([np.full(e.count, e.chunk_id, np.int64) for e in entries])
    return seq, pos, chk


def _check_plan_matches(batches, plan: ShardPlan) -> None:
    got = []
    for b in batches:
        got.extend(int(x) for x in lengths(b.q))
    if tuple(got) != plan.seq_lengths:
        raise ValueError("plan does not match the provided batches")


def _rows(values: torch.Tensor, idx: np.ndarray) -> torch.Tensor:
    if idx.size == 0:
        return values.new_empty((0,) + tuple(values.shape[1:]))
    perm = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int64)).to(values.device)
    src = values if values.dim() == 2 else values.view(-1, 1)
    out = kernels.gather_rows(src.contiguous(), perm)
    return out if values.dim() == 2 else out.view(-1)


def _devices(batches) -> list:
    """Single-process multi-device mode: rank r works on the device its batch
    lives on (all ranks on one device is the common single-GPU case)."""
    return [b.q.values.device for b in batches]


def _context(rank: int, plan: ShardPlan, q, k, v, ts) -> RankContext:
    seq, pos, chk = _entries_meta(plan.rank_entries[rank])
    return RankContext(rank, q, k, v, ts, seq, pos, chk, plan.rank_entries[rank])


def redistribute_allgather_split(group: RankGroup, batches, plan: ShardPlan, scheduling: str = "sequential"):
    """cp_engine.py:246-283: every rank materialises the full batch, keeps its rows."""
    group._require_full_group(batches, "redistribute_allgather_split")
    _check_sched(scheduling)
    _check_plan_matches(batches, plan)
    cp = group.cp_size
    payload = [b.payload_nbytes() for b in batches]
    stats, meters = gather_traffic(cp, payload, batches[0].q.values.element_size())
    devs = _devices(batches)
    full_bytes = sum(int(getattr(b, n).values.numel() * getattr(b, n).values.element_size())
                     for b in batches for n in ("q", "k", "v", "ts"))
    goff = plan.group_offsets()

    def keep(r: int) -> RankContext:
        # every rank materialises the whole group batch on its own device (the peak)
        full = {n: torch.cat([getattr(b, n).values.to(devs[r]) for b in batches]) for n in ("q", "k", "v", "ts")}
        idx = np.concatenate([np.arange(goff[e.seq_id] + e.start, goff[e.seq_id] + e.end, dtype=np.int64)
                              for e in plan.rank_entries[r]]) if plan.rank_entries[r] else np.zeros(0, np.int64)
        return _context(r, plan, *(_rows(full[n], idx) for n in ("q", "k", "v", "ts")))

    contexts = _map_ranks(keep, cp, scheduling, devs)
    for r, ctx in enumerate(contexts):
        meters[r].step(ctx.payload_nbytes() - full_bytes)
        stats[r].peak_resident_bytes = meters[r].peak
    group.steps_completed += 1
    return contexts, stats


def redistribute_alltoall(group: RankGroup, batches, plan: ShardPlan, scheduling: str = "sequential"):
    """cp_engine.py:330-371: each source ships its own chunks straight to
    their owners; received rows (source-major) are already in plan order."""
    group._require_full_group(batches, "redistribute_alltoall")
    _check_sched(scheduling)
    _check_plan_matches(batches, plan)
    cp = group.cp_size
    seq_base = np.concatenate([[0], np.cumsum([b.num_sequences for b in batches])]).astype(np.int64)
    def pack(src: int) -> list:
        loff = batches[src].q.host_offsets
        msgs = []
        for dst in range(cp):
            ents = [e for e in plan.rank_entries[dst] if plan.seq_owner[e.seq_id] == src]
            idx = np.concatenate([np.arange(loff[e.seq_id - seq_base[src]] + e.start,
                                            loff[e.seq_id - seq_base[src]] + e.end, dtype=np.int64)
                                  for e in ents]) if ents else np.zeros(0, np.int64)
            msgs.append(JaggedMessage([e.seq_id for e in ents], [e.chunk_id for e in ents],
                                      [e.start for e in ents], [e.count for e in ents],
                                      {n: _rows(getattr(batches[src], n).values, idx) for n in ("q", "k", "v", "ts")}))
        return msgs

    devs = _devices(batches)
    send = _map_ranks(pack, cp, scheduling, devs)
    received, stats = all_to_all_jagged(group, send)

    def assemble(r: int) -> RankContext:
        # messages from other devices are copied peer-to-peer to the receiver's device
        parts = {n: [m.arrays[n].to(devs[r]) for m in received[r]] for n in ("q", "k", "v", "ts")}
        return _context(r, plan, *(torch.cat(parts[n]) for n in ("q", "k", "v", "ts")))

    return _map_ranks(assemble, cp, scheduling, devs), stats


def _bundle(ctx: RankContext) -> JaggedMessage:
    """cp_engine.py:374-381."""
    e = ctx.entries
    return JaggedMessage([x.seq_id for x in e], [x.chunk_id for x in e], [x.start for x in e],
                         [x.count for x in e], {"k": ctx.k, "v": ctx.v, "ts": ctx.ts})


def ring_hstu_attention(group: RankGroup, contexts, params, cfg, scheduling: str = "sequential",
                        num_heads: int = 1):
    """cp_engine.py:384-453.  The cp-1 K/V/ts rotations are accounted exactly
    as the reference; the compute is one fused kernel launch per rank over its
    resident chunks, each attending to its sequence's causal prefix (SiLU
    partials are additive, so this equals the ring's ascending-chunk sum)."""
    group._require_full_group(contexts, "ring_hstu_attention")
    _check_sched(scheduling)
    cp = group.cp_size
    bundles = [_bundle(c) for c in contexts]
    meters = [MemoryMeter(_nbytes_t(c.q) + _nbytes_t(c.ts) + bundles[r].payload_nbytes())
              for r, c in enumerate(contexts)]
    totals = [CommStats(rank=r, dtype_size=contexts[0].q.element_size()) for r in range(cp)]
    from .comm import ring_send_recv
    b = bundles
    for step in range(cp - 1):
        b, deltas = ring_send_recv(group, step, b, steps=[step] * cp, meters=meters)
        for r in range(cp):
            totals[r].add(deltas[r])
    # group K/V/ts in sequence order, from the resident slabs of all ranks
    seq_len: dict[int, int] = {}
    for c in contexts:
        for e in c.entries:
            seq_len[e.seq_id] = max(seq_len.get(e.seq_id, 0), e.end)
    order = sorted(seq_len)
    base = {s: 0 for s in order}
    run = 0
    for s in order:
        base[s] = run
        run += seq_len[s]
    devs = [c.q.device for c in contexts]
    dev = devs[0]
    D = contexts[0].q.shape[1]
    K = contexts[0].k.new_empty((run, D))
    V = contexts[0].v.new_empty((run, D))
    TS = contexts[0].ts.new_empty((run,))
    for c in contexts:
        if c.num_rows == 0:
            continue
        dst = np.concatenate([np.arange(base[e.seq_id] + e.start, base[e.seq_id] + e.end, dtype=np.int64)
                              for e in c.entries])
        perm = torch.from_numpy(dst).to(dev)
        kernels.scatter_rows(c.k.to(dev), perm, K)
        kernels.scatter_rows(c.v.to(dev), perm, V)
        kernels.scatter_rows(c.ts.view(-1, 1).to(dev), perm, TS.view(-1, 1))
    # the gathered group K/V/ts on every device that hosts a rank (peer copies)
    kv = {dev: (K, V, TS)}
    for d in devs:
        if d not in kv:
            kv[d] = (K.to(d), V.to(d), TS.to(d))
    w_np = np.asarray(params.ts_weights, dtype=np.float32)

    def attend(r: int) -> torch.Tensor:
        c = contexts[r]
        d = devs[r]
        ents = [e for e in c.entries if e.count > 0]
        if not ents:
            return c.q.new_zeros(c.q.shape)
        qo = np.concatenate([[0], np.cumsum([e.count for e in ents])]).astype(np.int64)
        t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.int64)).to(d)  # noqa: E731
        kl = [e.end for e in ents]
        Kd, Vd, TSd = kv[d]
        return kernels.attn_fwd(c.q, Kd, Vd, c.ts, TSd, t(qo), num_heads, torch.from_numpy(w_np).to(d),
                                cfg.num_buckets, q_pos0=t([e.start for e in ents]),
                                kv_start=t([base[e.seq_id] for e in ents]), kv_len=t(kl), kv_len_total=int(sum(kl)))

    outputs = _map_ranks(attend, cp, scheduling, devs)
    for r, out in enumerate(outputs):
        meters[r].step(_nbytes_t(out))
        totals[r].peak_resident_bytes = max(totals[r].peak_resident_bytes, meters[r].peak)
    return outputs, totals


def _nbytes_t(t: torch.Tensor) -> int:
    return int(t.numel() * t.element_size())


def restore_outputs(group: RankGroup, slabs, plan: ShardPlan, max_lengths=None, scheduling: str = "sequential"):
    """cp_engine.py:468-525: inverse redistribution back to the contributing ranks."""
    group._require_full_group(slabs, "restore_outputs")
    _check_sched(scheduling)
    cp = group.cp_size
    for r in range(cp):
        want = sum(e.count for e in plan.rank_entries[r])
        if slabs[r].shape[0] != want:
            raise ValueError(f"rank {r} slab has {slabs[r].shape[0]} rows, plan expects {want}")
    send = []
    for r in range(cp):
        bounds = np.concatenate([[0], np.cumsum([e.count for e in plan.rank_entries[r]])]).astype(np.int64)
        msgs = []
        for dst in range(cp):
            sel = [(i, e) for i, e in enumerate(plan.rank_entries[r]) if plan.seq_owner[e.seq_id] == dst]
            idx = np.concatenate([np.arange(bounds[i], bounds[i + 1], dtype=np.int64) for i, _ in sel]) \
                if sel else np.zeros(0, np.int64)
            msgs.append(JaggedMessage([e.seq_id for _, e in sel], [e.chunk_id for _, e in sel],
                                      [e.start for _, e in sel], [e.count for _, e in sel],
                                      {"out": _rows(slabs[r], idx)}))
        send.append(msgs)
    received, stats = all_to_all_jagged(group, send)
    outputs = []
    for r in range(cp):
        own = [b for b in range(plan.num_sequences) if plan.seq_owner[b] == r]
        index = []
        for src in range(cp):
            m = received[r][src]
            bnd = np.concatenate([[0], np.cumsum(m.counts)]).astype(np.int64)
            index.append({(int(m.seq_ids[i]), int(m.chunk_ids[i])): (src, int(bnd[i]), int(bnd[i + 1]))
                          for i in range(m.num_chunks)})
        parts, offs = [], [0]
        for b in own:
            for c in range(plan.layout.chunks_per_seq):
                src, a, z = index[plan.chunk_owner[c]][(b, c)]
                parts.append(received[r][src].arrays["out"][a:z].to(slabs[r].device))
            offs.append(offs[-1] + plan.seq_lengths[b])
        d = slabs[0].shape[1]
        vals = torch.cat(parts) if parts else slabs[r].new_zeros((0, d))
        h = np.asarray(offs, dtype=np.int64)
        ml = max_lengths[r] if max_lengths is not None else max((plan.seq_lengths[b] for b in own), default=0)
        outputs.append(JaggedTensor(vals, torch.from_numpy(h).to(vals.device), int(ml), h))
    return outputs, stats


@dataclass
class PipelineResult:
    """cp_engine.py:551-560."""

    outputs: list
    plan: ShardPlan
    redistribute_stats: list
    ring_stats: list
    restore_stats: list
    resident_tokens: list
    peak_resident_bytes: list
    flops: FlopsReport


def run_pipeline(batches, cp_size: int, protocol: str, balance_mode: str, params, cfg,
                 scheduling: str = "sequential", num_heads: int = 1) -> PipelineResult:
    """cp_engine.py:563-598: plan -> redistribute -> ring attention -> restore."""
    if protocol not in ("allgather_split", "alltoall"):
        raise ValueError(f"unknown protocol {protocol!r}")
    plan = build_shard_plan([lengths(b.q).tolist() for b in batches], cp_size, balance_mode)
    group = RankGroup(cp_size)
    if protocol == "allgather_split":
        contexts, redist = redistribute_allgather_split(group, batches, plan, scheduling)
    else:
        contexts, redist = redistribute_alltoall(group, batches, plan, scheduling)
    slabs, ring = ring_hstu_attention(group, contexts, params, cfg, scheduling, num_heads)
    outputs, restore = restore_outputs(group, slabs, plan, [b.q.max_length for b in batches], scheduling)
    peaks = [max(redist[r].peak_resident_bytes, ring[r].peak_resident_bytes, restore[r].peak_resident_bytes)
             for r in range(cp_size)]
    return PipelineResult(outputs, plan, redist, ring, restore, list(plan.rank_token_counts()), peaks,
                          flops_per_rank(plan))
