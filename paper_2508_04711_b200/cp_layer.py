"""SPMD jagged context-parallel HSTU attention (one process per GPU).

This is the multi-GPU form of the reference pipeline ``run_pipeline``
(cp_engine.py:563-598: plan -> redistribute_alltoall -> ring_hstu_attention ->
restore_outputs), plus the backward pass the reference leaves out
(SPEC.md:390), over ``torch.distributed`` (NCCL on B200, gloo in CPU tests):

1. plan (cp_engine.py:105-147, exact integers from the C ABI): per-rank
   sequence lengths are all-gathered once per distinct batch shape and the
   balanced 2*CP mini-chunk plan is cached;
2. redistribution = one all-to-all (cp_engine.py:330-371): each rank packs its
   own sequences' chunks destination-major with the row-gather kernel; the
   received buffer is already in plan order (source-major == plan order);
3. KV exchange = all-gather of the resident K, V, ts slabs (cp_engine.py:
   384-453 rotates them in a ring; summing SiLU partials is order-free, so one
   gather + fused attention over the visible prefix gives the same result),
   issued on a side (communication) stream and overlapped with the local
   part: each resident chunk first attends to itself (its causal diagonal
   block, resident rows only) into an fp32 accumulator; once the gather lands,
   the gathered rows are re-ordered into sequence order and each chunk adds
   its remote part, the sequence prefix [0, chunk start) (all visible);
4. backward, mirrored: the remote part (chunk vs gathered prefix) first; its
   dK/dV partials for the whole group batch are reduced to their owners with
   reduce-scatter on the communication stream while the local part (chunk vs
   itself, dK/dV on resident rows) runs; dQ accumulates both parts in fp32;
   d_ts_weights is all-reduced;
5. restore = the inverse all-to-all (cp_engine.py:468-525).

Gradient semantics for DDP composition: ts_weights gradients are SUMMED over
the CP group here (every rank holds different tokens of the same batch);
average over data-parallel replicas only.
"""

from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .cp_engine import build_shard_plan


@dataclass
class CPPlan:
    """Host-side routing for one rank under one batch shape."""

    cp: int
    rank: int
    plan: object                 # ShardPlan (global)
    send_perm: np.ndarray        # local rows, destination-major (seq, chunk order)
    send_counts: list            # rows to each destination
    recv_counts: list            # rows from each source (== my resident rows per source)
    n_res: int                   # resident rows
    max_res: int                 # max resident rows over ranks (gather padding)
    res_counts: list             # resident rows of every rank
    seq_perm: np.ndarray         # group rows (sequence order) -> index in the padded gathered buffer
    q_offsets: np.ndarray        # resident segments (one per resident chunk)
    q_pos0: np.ndarray
    kv_start: np.ndarray
    kv_len: np.ndarray
    group_rows: int
    local_kv_start: np.ndarray   # overlap split: the rank's own rows (resident)
    local_kv_len: np.ndarray
    remote_kv_len: np.ndarray    # ... remote call A: [0, start of the rank's first chunk) in the gathered rows
    max_local: int = 0           # allgather_split: padded local rows per rank in the gathered batch
    split_perm: np.ndarray = None  # allgather_split: resident row -> index in the padded gathered batch
    local_q_pos0: np.ndarray = None  # overlap split: local segment q positions (later chunk: len of chunk r)
    remote2_kv_start: np.ndarray = None  # ... remote call B: the gap between the rank's two chunks
    remote2_kv_len: np.ndarray = None
    remote2_q_pos0: np.ndarray = None


def build_cp_plan(lengths_per_rank, cp: int, rank: int, balance_mode: str = "balanced_minichunk") -> CPPlan:
    plan = build_shard_plan(lengths_per_rank, cp, balance_mode)
    goff = plan.group_offsets()
    # local sequences of this rank: global ids [base, base + n_local)
    seq_base = int(np.sum([len(x) for x in lengths_per_rank[:rank]]))
    local_off = np.concatenate([[0], np.cumsum(lengths_per_rank[rank])]).astype(np.int64)
    # (1) pack order for redistribution: destination-major, plan order within
    send_rows, send_counts = [], []
    for dst in range(cp):
        n = 0
        for e in plan.rank_entries[dst]:
            if plan.seq_owner[e.seq_id] != rank:
                continue
            base = int(local_off[e.seq_id - seq_base])
            send_rows.append(np.arange(base + e.start, base + e.end, dtype=np.int64))
            n += e.count
        send_counts.append(n)
    send_perm = np.concatenate(send_rows) if send_rows else np.zeros(0, np.int64)
    # (2) receive counts per source (my plan entries, grouped by the contributing rank)
    recv_counts = [0] * cp
    for e in plan.rank_entries[rank]:
        recv_counts[plan.seq_owner[e.seq_id]] += e.count
    res_counts = list(plan.rank_token_counts())
    n_res, max_res = res_counts[rank], max(res_counts) if res_counts else 0
    # (3) sequence-order view of the padded, rank-major gathered buffer
    seq_perm = np.zeros(int(goff[-1]), dtype=np.int64)
    for r in range(cp):
        row = r * max_res
        for e in plan.rank_entries[r]:
            g0 = int(goff[e.seq_id])
            seq_perm[g0 + e.start:g0 + e.end] = np.arange(row, row + e.count, dtype=np.int64)
            row += e.count
    # (4) one attention segment per resident chunk: causal prefix [0, end) of its
    # sequence (non-overlapped form), and the overlapped split of the same work
    # (SURVEY §8(e)): LOCAL = what the rank's own rows cover -- chunk r against
    # itself, and chunk 2cp-1-r against [chunk r | itself], which are adjacent
    # resident rows (positions: chunk r at 0.., the later chunk at len_r..: the
    # causal mask is exact and the bias depends on timestamps only) -- and
    # REMOTE = the rest of the prefix in the gathered rows: [0, start of the
    # rank's first chunk) (call A) and, for a later chunk, the gap between the
    # rank's two chunks (call B; its own segment, all pairs visible, relative
    # positions exact by translation)
    qo, qp, ks, kl, lks, lkl, lqp = [0], [], [], [], [], [], []
    ra_len, rb_start, rb_len, rb_qp = [], [], [], []
    prev = None  # (seq_id, resident offset, entry) of the previous non-empty entry
    for e in plan.rank_entries[rank]:
        if e.count == 0:
            continue
        off = qo[-1]
        g0 = int(goff[e.seq_id])
        pair = prev is not None and prev[0] == e.seq_id
        if pair:
            _, poff, pe = prev
            lks.append(poff)
            lkl.append(pe.count + e.count)
            lqp.append(pe.count)
            ra_len.append(pe.start)
            rb_start.append(g0 + pe.end)
            rb_len.append(e.start - pe.end)
            rb_qp.append(e.start - pe.end)
        else:
            lks.append(off)
            lkl.append(e.count)
            lqp.append(0)
            ra_len.append(e.start)
            rb_start.append(g0)
            rb_len.append(0)
            rb_qp.append(0)
        prev = (e.seq_id, off, e)
        qo.append(off + e.count)
        qp.append(e.start)
        ks.append(g0)
        kl.append(e.end)
    # (5) allgather_split (cp_engine.py:246-283): every rank gathers all local
    # batches (rank-major, each padded to max_local rows) and keeps its plan rows
    local_tot = [int(sum(x)) for x in lengths_per_rank]
    max_local = max(local_tot) if local_tot else 0
    seq_local0 = np.zeros(len(plan.seq_owner), dtype=np.int64)  # first local row of each sequence
    nxt = [0] * cp
    for sid, (L, own) in enumerate(zip(plan.seq_lengths, plan.seq_owner)):
        seq_local0[sid] = nxt[own]
        nxt[own] += int(L)
    split_rows = [np.arange(e.start, e.end, dtype=np.int64) + plan.seq_owner[e.seq_id] * max_local +
                  seq_local0[e.seq_id] for e in plan.rank_entries[rank]]
    split_perm = np.concatenate(split_rows) if split_rows else np.zeros(0, np.int64)
    a64 = lambda x: np.asarray(x, np.int64)  # noqa: E731
    return CPPlan(cp, rank, plan, send_perm, send_counts, recv_counts, n_res, max_res, res_counts, seq_perm,
                  a64(qo), a64(qp), a64(ks), a64(kl), int(goff[-1]), a64(lks), a64(lkl), a64(ra_len), max_local,
                  split_perm, a64(lqp), a64(rb_start), a64(rb_len), a64(rb_qp))


class TorchComm:
    """The layer's collectives over a torch.distributed group (NCCL on B200:
    device tensors straight to the collective)."""

    def __init__(self, group, device=None):
        self.group = group
        self.size = dist.get_world_size(group)
        self.device = device

    def _dev(self, like=None):
        if self.device is not None:
            return self.device
        if like is not None:
            return like.device
        return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(self.group) == "nccl" \
            else torch.device("cpu")

    MAX_SEQS = 16384  # per-rank sequence capacity of the length exchange

    def lengths_start(self, local_lengths):
        """Start the length exchange: ONE all-gather of a fixed-capacity
        [count, lengths...] int64 row per rank (no count round, no .item()),
        then an asynchronous copy into pinned host memory; returns a handle for
        ``lengths_finish``.  The host waits only when the plan is needed
        (asynchronous offsets, sync delayed), so a training loop
        can start the next batch's exchange before this step's compute ends
        (CPAttention.prefetch_plan)."""
        loc = np.asarray(local_lengths, dtype=np.int64)
        if loc.size > self.MAX_SEQS:
            raise ValueError(f"{loc.size} sequences exceed the length-exchange capacity {self.MAX_SEQS}")
        dev = self._dev()
        row = np.zeros(self.MAX_SEQS + 1, dtype=np.int64)
        row[0] = loc.size
        row[1:1 + loc.size] = loc
        t_row = torch.from_numpy(row)
        # (pinned: a pageable host->device copy makes the host wait for the stream first)
        send = t_row.pin_memory().to(dev, non_blocking=True) if dev.type == "cuda" else t_row
        full = torch.empty((self.size, self.MAX_SEQS + 1), dtype=torch.int64, device=dev)
        self._all_gather(list(full.unbind(0)), send)
        if dev.type == "cuda":
            host = torch.empty(full.shape, dtype=torch.int64, pin_memory=True)
            host.copy_(full, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            return host, ev
        return full, None

    @staticmethod
    def lengths_finish(handle) -> tuple:
        host, ev = handle
        if ev is not None:
            ev.synchronize()
        h = host.numpy()
        return tuple(tuple(int(v) for v in r[1:1 + int(r[0])]) for r in h)

    def all_gather_lengths(self, local_lengths) -> tuple:
        """Every rank's sequence lengths, identical on all ranks."""
        return self.lengths_finish(self.lengths_start(local_lengths))

    def _all_gather(self, outs, x):
        dist.all_gather(outs, x, group=self.group)

    def all_to_all(self, out, send, out_splits, in_splits):
        dist.all_to_all_single(out, send, list(out_splits), list(in_splits), group=self.group)

    def all_gather_into(self, full, x):
        dist.all_gather_into_tensor(full, x, group=self.group)

    def reduce_scatter(self, out, full):
        dist.reduce_scatter_tensor(out, full, group=self.group)

    def all_reduce(self, x):
        dist.all_reduce(x, group=self.group)


class HostStagedComm(TorchComm):
    """Same collectives for a CPU (gloo) group with device tensors: each call
    stages through host memory.  Lets several processes that share one GPU run
    the real CUDA layer (tests), with no kernel waiting on another process."""

    def _dev(self, like=None):
        return torch.device("cpu")

    @staticmethod
    def _host(x):
        return x.detach().to("cpu")

    def _all_gather(self, outs, x):
        dist.all_gather(outs, self._host(x), group=self.group)

    def all_to_all(self, out, send, out_splits, in_splits):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(h, self._host(send), list(out_splits), list(in_splits), group=self.group)
        out.copy_(h)

    def all_gather_into(self, full, x):
        h = torch.empty(full.shape, dtype=full.dtype)
        dist.all_gather_into_tensor(h, self._host(x), group=self.group)
        full.copy_(h)

    def reduce_scatter(self, out, full):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.reduce_scatter_tensor(h, self._host(full), group=self.group)
        out.copy_(h)

    def all_reduce(self, x):
        h = self._host(x).clone()
        dist.all_reduce(h, group=self.group)
        x.copy_(h)


class GpuBackend:
    """Compute pieces on the B200 kernels (libjh_hstu.so)."""

    def __init__(self):
        from . import kernels
        self.k = kernels

    def gather(self, src, perm):
        return self.k.gather_rows(src, perm)

    def scatter(self, src, perm, out):
        return self.k.scatter_rows(src, perm, out)

    def fwd(self, q, k, v, ts_q, ts_k, segs, H, w, nb):
        qo, qp, ks, kl, kvt = segs[:5]
        return self.k.attn_fwd(q, k, v, ts_q, ts_k, qo, H, w, nb, q_pos0=qp, kv_start=ks, kv_len=kl,
                               kv_len_total=kvt)

    def fwd_partial(self, q, k, v, ts_q, ts_k, segs, H, w, nb, acc, accumulate):
        qo, qp, ks, kl, kvt = segs[:5]
        self.k.attn_fwd(q, k, v, ts_q, ts_k, qo, H, w, nb, q_pos0=qp, kv_start=ks, kv_len=kl, kv_len_total=kvt,
                        out_accum=acc, accumulate=accumulate)

    def comm_stream(self, device):
        if device.type != "cuda":
            return None
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream(device=device)
        return self._comm

    def bwd(self, q, k, v, ts_q, ts_k, segs, g, H, w, nb):
        qo, qp, ks, kl, kvt = segs[:5]
        dq, dk, dv, dw, _ = self.k.attn_bwd(q, k, v, ts_q, ts_k, qo, g, H, w, nb, q_pos0=qp, kv_start=ks,
                                            kv_len=kl, kv_len_total=kvt, accumulate_dkv=True, seg_host=segs[6])
        return dq, dk, dv, dw

    def bwd_partial(self, q, k, v, ts_q, ts_k, segs, g, H, w, nb, dq_acc, dkv=None):
        qo, qp, ks, kl, kvt = segs[:5]
        _, dk, dv, dw, _ = self.k.attn_bwd(q, k, v, ts_q, ts_k, qo, g, H, w, nb, q_pos0=qp, kv_start=ks, kv_len=kl,
                                           kv_len_total=kvt, accumulate_dkv=True, seg_host=segs[6],
                                           dq_accum=dq_acc, dkv_accum=dkv)
        return dk, dv, dw


class LoopbackComm:
    """One process standing in for rank ``rank`` of a CP group of ``size``
    ranks, communication EXCLUDED: every collective returns a correctly sized
    buffer filled from local data (the other ranks' K/V are replicas of this
    rank's, so values are meaningless but shapes, memory and kernel work are
    exactly one rank's).  Used by the bench's per-rank max-length probe
    (bench.py --cp-probe), the measured analogue of the reference's modeled
    per-rank footprint (harness.py:308-374)."""

    def __init__(self, size: int, rank: int = 0, peer_lengths=None):
        self.size, self.rank = int(size), int(rank)
        self.peer_lengths = peer_lengths  # callable rank -> lengths of that rank's local batch

    def all_gather_lengths(self, local_lengths) -> tuple:
        loc = tuple(int(x) for x in local_lengths)
        if self.peer_lengths is None:
            return tuple(loc for _ in range(self.size))
        return tuple(loc if r == self.rank else tuple(int(x) for x in self.peer_lengths(r))
                     for r in range(self.size))

    def all_to_all(self, out, send, out_splits, in_splits):
        out.zero_()

    def all_gather_into(self, full, x):
        full.view((self.size,) + tuple(x.shape)).copy_(x.unsqueeze(0).expand((self.size,) + tuple(x.shape)))

    def reduce_scatter(self, out, full):
        out.copy_(full.view((self.size,) + tuple(out.shape))[self.rank])

    def all_reduce(self, x):
        pass


class CPAttention:
    """Context-parallel jagged HSTU attention over a process group (or, with
    ``group=None``, over the topology of ``comm``: a LoopbackComm probe)."""

    def __init__(self, group, num_heads: int, num_buckets: int = 16, balance_mode: str = "balanced_minichunk",
                 backend=None, overlap: bool = True, comm=None, max_plans: int = 64, retain_kv: bool = False,
                 protocol: str = "alltoall", measure: bool = False):
        self.group = group
        if group is None:
            if comm is None or not hasattr(comm, "size"):
                raise ValueError("group=None needs a comm that carries its topology (LoopbackComm)")
            self.cp, self.rank = comm.size, comm.rank
        else:
            self.cp = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        self.comm = comm if comm is not None else TorchComm(group)
        self.max_plans = int(max_plans)
        self.H = num_heads
        self.nb = num_buckets
        self.mode = balance_mode
        self.be = backend if backend is not None else GpuBackend()
        self.overlap = overlap and hasattr(self.be, "fwd_partial") and hasattr(self.be, "bwd_partial")
        self._plans: "OrderedDict" = OrderedDict()
        self._pending = None
        # exchange timing (CUDA events; exchange_report) -- off by default
        self.meter = {"coll": [], "join": []} if measure else None
        self._on_cuda = isinstance(self.be, GpuBackend)
        if protocol not in ("alltoall", "allgather_split"):
            raise ValueError(f"unknown protocol {protocol!r}")
        self.protocol = protocol
        # keep the gathered group K/V/ts between forward and backward (one fewer
        # all-gather per layer, O(group rows) memory) or re-gather them
        self.retain_kv = bool(retain_kv)

    # ---------------------------------------------------------------- plan
    def prefetch_plan(self, local_lengths) -> None:
        """Start the length exchange of a FUTURE step (e.g. the next batch,
        right after this step's forward is enqueued); the matching
        ``plan_for`` then only waits for a copy that finished long ago.  Every
        rank must prefetch at the same point (it is a collective)."""
        if hasattr(self.comm, "lengths_start"):
            loc = tuple(int(x) for x in local_lengths)
            self._pending = (loc, self.comm.lengths_start(list(loc)))

    def plan_for(self, local_lengths, device) -> tuple[CPPlan, dict]:
        """Every rank's lengths are all-gathered EVERY step and the plan cache is
        keyed on that global tuple, so all ranks make the same hit / miss /
        eviction decision (LRU over identical key sequences) and enter the same
        collectives."""
        loc = tuple(int(x) for x in local_lengths)
        pend = self._pending
        self._pending = None
        if pend is not None and pend[0] == loc:
            key = self.comm.lengths_finish(pend[1])
        else:
            key = self.comm.all_gather_lengths(list(loc))
        if key in self._plans:
            self._plans.move_to_end(key)
            return self._plans[key]
        p = build_cp_plan([list(x) for x in key], self.cp, self.rank, self.mode)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        dev = {"send_perm": t(p.send_perm), "seq_perm": t(p.seq_perm), "split_perm": t(p.split_perm),
               # (q_offsets, q_pos0, kv_start, kv_len, kv total, max kv,
               #  host (q_offsets, q_pos0, kv_len, kv_start): exact dS sizing + the windowed long-L backward)
               "segs": (t(p.q_offsets), t(p.q_pos0), t(p.kv_start), t(p.kv_len), int(p.kv_len.sum()),
                        int(p.kv_len.max(initial=0)), (p.q_offsets, p.q_pos0, p.kv_len, p.kv_start)),
               "local_segs": (t(p.q_offsets), t(p.local_q_pos0), t(p.local_kv_start),
                              t(p.local_kv_len), int(p.local_kv_len.sum()), int(p.local_kv_len.max(initial=0)),
                              (p.q_offsets, p.local_q_pos0, p.local_kv_len, p.local_kv_start)),
               "remote_segs": (t(p.q_offsets), t(p.q_pos0), t(p.kv_start), t(p.remote_kv_len),
                               int(p.remote_kv_len.sum()), int(p.remote_kv_len.max(initial=0)),
                               (p.q_offsets, p.q_pos0, p.remote_kv_len, p.kv_start))}
        if int(p.remote2_kv_len.sum()) > 0:  # remote call B (balanced mode: later chunks' gaps)
            dev["remote2_segs"] = (t(p.q_offsets), t(p.remote2_q_pos0), t(p.remote2_kv_start), t(p.remote2_kv_len),
                                   int(p.remote2_kv_len.sum()), int(p.remote2_kv_len.max(initial=0)),
                                   (p.q_offsets, p.remote2_q_pos0, p.remote2_kv_len, p.remote2_kv_start))
        self._plans[key] = (p, dev)
        while len(self._plans) > self.max_plans:
            self._plans.popitem(last=False)
        return self._plans[key]

    # ---------------------------------------------------------- collectives
    def _timed(self, name, nbytes, fn):
        """Run one collective; with ``measure`` on a CUDA stream, CUDA events
        bracket it on the stream it is issued on (exchange_report)."""
        if self.meter is None or not torch.cuda.is_available() or not self._on_cuda:
            return fn()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        r = fn()
        e1.record(s)
        self.meter["coll"].append((name, int(nbytes), e0, e1))
        return r

    def exchange_report(self, reset: bool = True) -> dict:
        """Per-collective totals since the last report: bytes (the collective's
        output buffer on this rank), device ms, GB/s against NVLink 5 (900 GB/s
        per direction), and the EXPOSED time -- how long the main stream waited
        for the communication stream (the part the overlap did not hide)."""
        if self.meter is None:
            return {}
        torch.cuda.synchronize()
        out = {}
        for name, nb, e0, e1 in self.meter["coll"]:
            d = out.setdefault(name, {"calls": 0, "bytes": 0, "ms": 0.0})
            d["calls"] += 1
            d["bytes"] += nb
            d["ms"] += e0.elapsed_time(e1)
        for d in out.values():
            d["GB_s"] = d["bytes"] / max(d["ms"], 1e-9) / 1e6
            d["frac_nvlink_900"] = d["GB_s"] / 900.0
        exposed = sum(max(0.0, a.elapsed_time(b)) for a, b in self.meter["join"])
        rep = {"collectives": out, "exposed_ms": exposed, "joins": len(self.meter["join"])}
        if reset:
            self.meter = {"coll": [], "join": []}
        return rep

    def _a2a_rows(self, send, send_counts, recv_counts):
        out = send.new_empty((int(sum(recv_counts)),) + tuple(send.shape[1:]))
        self._timed("all_to_all", out.numel() * out.element_size(),
                    lambda: self.comm.all_to_all(out, send, recv_counts, send_counts))
        return out

    def _redistribute(self, x, p, dev):
        """local rows -> resident rows in plan order: one all-to-all of the
        destination-packed rows (cp_engine.py:330-371), or with
        protocol="allgather_split" the reference's baseline -- gather every
        rank's whole local batch, keep the plan rows (cp_engine.py:246-283;
        peak = the full group batch on every rank)."""
        if self.protocol == "allgather_split":
            # (padding rows are gathered but never selected by split_perm: left uninitialised)
            pad = x.new_empty((p.max_local,) + tuple(x.shape[1:]))
            pad[: x.shape[0]] = x
            full = x.new_empty((self.cp * p.max_local,) + tuple(x.shape[1:]))
            self._timed("allgather_split", full.numel() * full.element_size(),
                        lambda: self.comm.all_gather_into(full, pad))
            return self.be.gather(full, dev["split_perm"])
        return self._a2a_rows(self.be.gather(x, dev["send_perm"]), p.send_counts, p.recv_counts)

    def _restore(self, x_res, p, dev, n_local):
        """resident rows -> local rows (cp_engine.py:468-525)."""
        back = self._a2a_rows(x_res, p.recv_counts, p.send_counts)
        out = x_res.new_empty((n_local,) + tuple(x_res.shape[1:]))
        return self.be.scatter(back, dev["send_perm"], out)

    def _gather_seq(self, x_res, p, dev):
        """resident slabs of all ranks -> group rows in sequence order."""
        pad = x_res.new_empty((p.max_res,) + tuple(x_res.shape[1:]))  # (padding never selected by seq_perm)
        pad[: p.n_res] = x_res
        full = x_res.new_empty((self.cp * p.max_res,) + tuple(x_res.shape[1:]))
        self._timed("kv_all_gather", full.numel() * full.element_size(), lambda: self.comm.all_gather_into(full, pad))
        return self.be.gather(full, dev["seq_perm"])

    def _reduce_to_owner(self, x_seq, p, dev):
        """sum of per-rank partials over group rows (sequence order) -> my resident rows."""
        # every owner's real rows are written by the scatter; the padding rows of
        # each owner's slice are reduced too but sliced off below: no zero fill
        full = x_seq.new_empty((self.cp * p.max_res,) + tuple(x_seq.shape[1:]))
        self.be.scatter(x_seq, dev["seq_perm"], full)
        mine = x_seq.new_empty((p.max_res,) + tuple(x_seq.shape[1:]))
        self._timed("dkv_reduce_scatter", full.numel() * full.element_size(),
                    lambda: self.comm.reduce_scatter(mine, full))
        return mine[: p.n_res]

    # --------------------------------------------------------------- passes
    def redistribute(self, x, p, dev):
        """Public form of the batch -> sequence sharding (any trailing shape)."""
        return self._redistribute(x, p, dev)

    def restore(self, x_r, p, dev, n_local):
        return self._restore(x_r, p, dev, n_local)

    def forward(self, q, k, v, ts, local_lengths, w):
        """Local (batch-sharded) q, k, v, ts -> local attention output.
        Returns (out_local, ctx) where ctx feeds ``backward``."""
        p, dev = self.plan_for(local_lengths, q.device)
        q_r, k_r, v_r = (self._redistribute(x, p, dev) for x in (q, k, v))
        ts_r = self._redistribute(ts.view(-1, 1), p, dev).view(-1)
        o_r, rctx = self.attend(q_r, k_r, v_r, ts_r, p, dev, w)
        out = self._restore(o_r, p, dev, q.shape[0])
        return out, (rctx, q.shape[0])

    def attend(self, q_r, k_r, v_r, ts_r, p, dev, w):
        """Attention on RESIDENT rows (plan order; the sharded activations of a
        CP stack stay in this layout across layers): KV exchange + fused
        kernels.  Returns (o_r, ctx) for ``attend_backward``."""
        if not self.overlap:
            k_s, v_s = self._gather_seq(k_r, p, dev), self._gather_seq(v_r, p, dev)
            ts_s = self._gather_seq(ts_r.view(-1, 1), p, dev).view(-1)
            o_r = self.be.fwd(q_r, k_s, v_s, ts_r, ts_s, dev["segs"], self.H, w, self.nb)
        else:
            k_s, v_s, ts_s, o_r = self._forward_overlapped(q_r, k_r, v_r, ts_r, p, dev, w)
        if not self.retain_kv:  # re-gathered by the backward: O(resident) memory between the passes
            k_s = v_s = ts_s = None
        return o_r, (p, dev, q_r, k_s, v_s, ts_r, ts_s, k_r, v_r)

    def _forward_overlapped(self, q_r, k_r, v_r, ts_r, p, dev, w):
        """KV all-gather on the communication stream while each resident chunk
        attends to itself; then the remote prefix is added (SiLU partials are
        additive, attention.py:151-184 / cp_engine.py:441-450)."""
        main = torch.cuda.current_stream(q_r.device) if q_r.is_cuda else None
        comm = self.be.comm_stream(q_r.device) if hasattr(self.be, "comm_stream") else None
        k_s, v_s, ts_s = self._gather_kv_async(k_r, v_r, ts_r, p, dev, main, comm)
        acc_dt = torch.float32 if q_r.dtype in (torch.bfloat16, torch.float16) else q_r.dtype
        acc = torch.empty(q_r.shape, dtype=acc_dt, device=q_r.device)
        self.be.fwd_partial(q_r, k_r, v_r, ts_r, ts_r, dev["local_segs"], self.H, w, self.nb, acc, False)
        self._join(main, comm, (k_s, v_s, ts_s))
        self.be.fwd_partial(q_r, k_s, v_s, ts_r, ts_s, dev["remote_segs"], self.H, w, self.nb, acc, True)
        if "remote2_segs" in dev:
            self.be.fwd_partial(q_r, k_s, v_s, ts_r, ts_s, dev["remote2_segs"], self.H, w, self.nb, acc, True)
        return k_s, v_s, ts_s, acc.to(q_r.dtype)

    def _gather_kv_async(self, k_r, v_r, ts_r, p, dev, main, comm):
        if comm is not None:
            comm.wait_stream(main)
            for x in (k_r, v_r, ts_r):
                x.record_stream(comm)
            with torch.cuda.stream(comm):
                k_s, v_s = self._gather_seq(k_r, p, dev), self._gather_seq(v_r, p, dev)
                ts_s = self._gather_seq(ts_r.view(-1, 1), p, dev).view(-1)
        else:
            k_s, v_s = self._gather_seq(k_r, p, dev), self._gather_seq(v_r, p, dev)
            ts_s = self._gather_seq(ts_r.view(-1, 1), p, dev).view(-1)
        return k_s, v_s, ts_s

    def _join(self, main, comm, tensors):
        if comm is not None:
            if self.meter is not None:
                need, done = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                need.record(main)
                done.record(comm)
                self.meter["join"].append((need, done))
            main.wait_stream(comm)
            for x in tensors:
                x.record_stream(main)

    def backward(self, ctx, g, w):
        """Upstream gradient (local rows) -> (dq, dk, dv local; d_ts_weights summed over CP)."""
        rctx, n_local = ctx
        p, dev = rctx[0], rctx[1]
        g_r = self._redistribute(g, p, dev)
        dq_r, dk_r, dv_r, dw = self.attend_backward(rctx, g_r, w)
        dq = self._restore(dq_r, p, dev, n_local)
        dk = self._restore(dk_r, p, dev, n_local)
        dv = self._restore(dv_r, p, dev, n_local)
        return dq, dk, dv, dw

    def attend_backward(self, rctx, g_r, w):
        """Resident-row backward: (dq_r, dk_r, dv_r, d_ts_weights summed over CP)."""
        p, dev, q_r, k_s, v_s, ts_r, ts_s, k_r, v_r = rctx
        if not self.overlap:
            if k_s is None:
                k_s, v_s = self._gather_seq(k_r, p, dev), self._gather_seq(v_r, p, dev)
                ts_s = self._gather_seq(ts_r.view(-1, 1), p, dev).view(-1)
            dq_r, dk_s, dv_s, dw = self.be.bwd(q_r, k_s, v_s, ts_r, ts_s, dev["segs"], g_r, self.H, w, self.nb)
            dk_r = self._reduce_to_owner(dk_s, p, dev).to(q_r.dtype)
            dv_r = self._reduce_to_owner(dv_s, p, dev).to(q_r.dtype)
        elif k_s is None:
            dq_r, dk_r, dv_r, dw = self._backward_regather(q_r, k_r, v_r, ts_r, g_r, p, dev, w)
        else:
            dq_r, dk_r, dv_r, dw = self._backward_overlapped(q_r, k_r, v_r, k_s, v_s, ts_r, ts_s, g_r, p, dev, w)
        self._timed("d_w_all_reduce", dw.numel() * dw.element_size(), lambda: self.comm.all_reduce(dw))
        return dq_r, dk_r, dv_r, dw

    def _remote_bwd(self, q_r, k_s, v_s, ts_r, ts_s, g_r, dev, w, dq_acc):
        """Remote calls A (and B): dK/dV partials over the gathered rows, dq added."""
        dk_s, dv_s, dw = self.be.bwd_partial(q_r, k_s, v_s, ts_r, ts_s, dev["remote_segs"], g_r, self.H, w, self.nb,
                                             dq_acc)
        if "remote2_segs" in dev:  # call B adds into call A's group-size fp32 partials (no third buffer)
            _, _, dw2 = self.be.bwd_partial(q_r, k_s, v_s, ts_r, ts_s, dev["remote2_segs"], g_r, self.H, w,
                                            self.nb, dq_acc, dkv=(dk_s, dv_s))
            dw = dw + dw2
        return dk_s, dv_s, dw

    def _backward_regather(self, q_r, k_r, v_r, ts_r, g_r, p, dev, w):
        """K/V were not kept: re-gather them on the communication stream while
        the local part (chunk vs itself) computes, then the remote part; its
        dK/dV partials are reduced to the owners afterwards."""
        acc_dt = torch.float32 if q_r.dtype in (torch.bfloat16, torch.float16) else q_r.dtype
        main = torch.cuda.current_stream(q_r.device) if q_r.is_cuda else None
        comm = self.be.comm_stream(q_r.device) if hasattr(self.be, "comm_stream") else None
        k_s, v_s, ts_s = self._gather_kv_async(k_r, v_r, ts_r, p, dev, main, comm)
        dq_acc = torch.zeros(q_r.shape, dtype=acc_dt, device=q_r.device)
        dk_l, dv_l, dw_l = self.be.bwd_partial(q_r, k_r, v_r, ts_r, ts_r, dev["local_segs"], g_r, self.H, w, self.nb,
                                               dq_acc)
        self._join(main, comm, (k_s, v_s, ts_s))
        dk_s, dv_s, dw = self._remote_bwd(q_r, k_s, v_s, ts_r, ts_s, g_r, dev, w, dq_acc)
        dk_red, dv_red = self._reduce_to_owner(dk_s, p, dev), self._reduce_to_owner(dv_s, p, dev)
        return dq_acc.to(q_r.dtype), (dk_red + dk_l).to(q_r.dtype), (dv_red + dv_l).to(q_r.dtype), dw + dw_l

    def _backward_overlapped(self, q_r, k_r, v_r, k_s, v_s, ts_r, ts_s, g_r, p, dev, w):
        """Remote part first; its dK/dV reduce-scatter to the owners runs on the
        communication stream while the local (chunk vs itself) part computes."""
        acc_dt = torch.float32 if q_r.dtype in (torch.bfloat16, torch.float16) else q_r.dtype
        dq_acc = torch.zeros(q_r.shape, dtype=acc_dt, device=q_r.device)
        dk_s, dv_s, dw = self._remote_bwd(q_r, k_s, v_s, ts_r, ts_s, g_r, dev, w, dq_acc)
        main = torch.cuda.current_stream(q_r.device) if q_r.is_cuda else None
        comm = self.be.comm_stream(q_r.device) if hasattr(self.be, "comm_stream") else None
        if comm is not None:
            comm.wait_stream(main)
            for x in (dk_s, dv_s):
                x.record_stream(comm)
            with torch.cuda.stream(comm):
                dk_red, dv_red = self._reduce_to_owner(dk_s, p, dev), self._reduce_to_owner(dv_s, p, dev)
        else:
            dk_red, dv_red = self._reduce_to_owner(dk_s, p, dev), self._reduce_to_owner(dv_s, p, dev)
        dk_l, dv_l, dw_l = self.be.bwd_partial(q_r, k_r, v_r, ts_r, ts_r, dev["local_segs"], g_r, self.H, w, self.nb,
                                               dq_acc)
        self._join(main, comm, (dk_red, dv_red))
        dk_r = (dk_red + dk_l).to(q_r.dtype)
        dv_r = (dv_red + dv_l).to(q_r.dtype)
        return dq_acc.to(q_r.dtype), dk_r, dv_r, dw + dw_l

    def bench_step(self, q, k, v, ts, local_offsets, g, w):
        lengths = np.diff(np.asarray(local_offsets))

        def step(prof=None):
            _, ctx = self.forward(q, k, v, ts, lengths, w)
            # the next step's length exchange starts now (a training loop would
            # pass its next batch's lengths), so plan_for never waits for it
            self.prefetch_plan(lengths)
            return self.backward(ctx, g, w)

        return step


class _CPAttentionFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, ts_weights, ts, lengths, layer):
        out, c = layer.forward(q, k, v, ts, lengths, ts_weights)
        ctx.c, ctx.layer = c, layer
        ctx.save_for_backward(ts_weights)
        return out

    @staticmethod
    def backward(ctx, g):
        (w,) = ctx.saved_tensors
        dq, dk, dv, dw = ctx.layer.backward(ctx.c, g.to(ctx.c[0][2].dtype).contiguous(), w)
        return dq, dk, dv, dw.to(w.dtype), None, None, None


class _CPResidentAttentionFn(torch.autograd.Function):
    """Attention over resident rows (plan order) -- the per-layer op of a CP
    stack whose activations stay sequence-sharded between layers."""

    @staticmethod
    def forward(ctx, q_r, k_r, v_r, ts_weights, ts_r, layer, plan):
        p, dev = plan
        o_r, rctx = layer.attend(q_r, k_r, v_r, ts_r, p, dev, ts_weights)
        ctx.rctx, ctx.layer = rctx, layer
        ctx.save_for_backward(ts_weights)
        return o_r

    @staticmethod
    def backward(ctx, g_r):
        (w,) = ctx.saved_tensors
        dq, dk, dv, dw = ctx.layer.attend_backward(ctx.rctx, g_r.to(ctx.rctx[2].dtype).contiguous(), w)
        ctx.rctx = None
        return dq, dk, dv, dw.to(w.dtype), None, None, None


class _ShardFn(torch.autograd.Function):
    """local rows -> resident rows (the all-to-all); its gradient is the inverse."""

    @staticmethod
    def forward(ctx, x, layer, plan, n_local):
        ctx.layer, ctx.plan, ctx.n_local = layer, plan, n_local
        return layer.redistribute(x, *plan)

    @staticmethod
    def backward(ctx, g):
        return ctx.layer.restore(g.contiguous(), *ctx.plan, ctx.n_local), None, None, None


class _UnshardFn(torch.autograd.Function):
    """resident rows -> local rows (restore_outputs); its gradient is the forward a2a."""

    @staticmethod
    def forward(ctx, x_r, layer, plan, n_local):
        ctx.layer, ctx.plan = layer, plan
        return layer.restore(x_r, *plan, n_local)

    @staticmethod
    def backward(ctx, g):
        return ctx.layer.redistribute(g.contiguous(), *ctx.plan), None, None, None


def cp_resident_attention(layer: CPAttention, plan, q_r, k_r, v_r, ts_r, ts_weights):
    return _CPResidentAttentionFn.apply(q_r, k_r, v_r, ts_weights, ts_r, layer, plan)


def cp_shard(layer: CPAttention, plan, x, n_local: int):
    return _ShardFn.apply(x, layer, plan, n_local)


def cp_unshard(layer: CPAttention, plan, x_r, n_local: int):
    return _UnshardFn.apply(x_r, layer, plan, n_local)


def cp_hstu_attention(layer: CPAttention, q, k, v, ts, local_lengths, ts_weights):
    """Differentiable CP attention (gradients to q, k, v and ts_weights)."""
    return _CPAttentionFn.apply(q, k, v, ts_weights, ts, np.asarray(local_lengths), layer)


# ------------------------------------------------------- hybrid CP x DP (C5)

def make_cp_dp_groups(cp_size: int, backend=None):
    """Process groups of a hybrid CP x DP layout:
    rank = dp_index * cp_size + cp_index, CP groups are consecutive ranks
    ({0..cp-1}, {cp..2cp-1}, ...), DP groups stride by cp_size ({0, cp, ...},
    {1, cp+1, ...}).  Every rank creates every group (torch.distributed
    requires the same new_group call sequence on all ranks).  Returns
    (cp_group, dp_group, cp_index, dp_index)."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    if cp_size < 1 or world % cp_size:
        raise ValueError(f"world size {world} is not a multiple of cp_size {cp_size}")
    dp_size = world // cp_size
    cp_group = dp_group = None
    for d in range(dp_size):
        g = dist.new_group(list(range(d * cp_size, (d + 1) * cp_size)), backend=backend)
        if rank // cp_size == d:
            cp_group = g
    for c in range(cp_size):
        g = dist.new_group(list(range(c, world, cp_size)), backend=backend)
        if rank % cp_size == c:
            dp_group = g
    return cp_group, dp_group, rank % cp_size, rank // cp_size


class CPJaggedHSTUAttention(torch.nn.Module):
    """The attention layer sharded along the sequence by jagged CP: learnable
    ts_weights around ``cp_hstu_attention``.  Composes with DDP over the DP
    group: CPAttention's backward SUMS the ts_weights gradient over the CP
    group (its ranks hold different tokens of one batch); wrapping this module
    in ``DistributedDataParallel(process_group=dp_group)`` then AVERAGES it
    over the data-parallel replicas -- the rule of SURVEY §7 hard part 6."""

    def __init__(self, cp_group, num_heads: int, num_buckets: int = 16, balance_mode: str = "balanced_minichunk",
                 seed: int = 0, backend=None, comm=None, overlap: bool = True, weights=None):
        super().__init__()
        if weights is None:
            from .attention import BiasConfig, BiasParams
            weights = BiasParams.normal_init(BiasConfig(num_buckets), seed).ts_weights
        self.ts_weights = torch.nn.Parameter(torch.as_tensor(np.asarray(weights, dtype=np.float32)).clone())
        self.cp = CPAttention(cp_group, num_heads, num_buckets, balance_mode, backend=backend, overlap=overlap,
                              comm=comm)

    def forward(self, q, k, v, ts, local_lengths):
        return cp_hstu_attention(self.cp, q, k, v, ts, local_lengths, self.ts_weights)
