"""Synthetic jagged batches, the error metric and the experiment / sweep
reports (mirror of ``jaggedcp/harness.py``: harness.py:52-368).

``gen_synthetic_batch`` draws from the same numpy RNG stream as the
reference (``default_rng([seed, rank])``: lengths, q, k, v, starts, gaps in
that order), so a config produces the reference's exact inputs; values are
then rounded to bf16 on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .attention import BiasConfig, BiasParams
from .jagged import new_int_series, new_jagged

PROTOCOLS = ("allgather_split", "alltoall")
LENGTH_DISTS = ("uniform", "lognormal")
SCHEDULINGS = ("sequential", "threaded")
MAX_TS_GAP_SECONDS = 1_000_000
DTYPE_SIZES = {"bf16": 2, "f32": 4, "f64": 8}

# harness.py:45-49 (same text: the report's accounting is the reference's)
ACCOUNTING_NOTE = (
    "residency counts value payloads (q/k/v/ts and outputs) in bytes; headers are "
    "tallied separately; gathers retain sent data while all-to-all relinquishes it; "
    "memory_reduction_ratio compares worst-rank redistribution peaks of the two protocols"
)


@dataclass(frozen=True)
class ExperimentConfig:
    """harness.py:52-95 (+ num_heads)."""

    cp_size: int = 2
    batch_size: int = 2
    length_dist: str = "uniform"
    min_len: int = 1
    max_len: int = 32
    lognorm_mu: float = 3.0
    lognorm_sigma: float = 0.8
    max_length: int = 128
    embed_dim: int = 8
    num_buckets: int = 16
    dtype: str = "bf16"
    protocol: str = "alltoall"
    balance_mode: str = "balanced_minichunk"
    seed: int = 0
    num_heads: int = 1

    def __post_init__(self) -> None:
        if self.cp_size < 1:
            raise ValueError("cp_size must be >= 1")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.length_dist not in LENGTH_DISTS:
            raise ValueError(f"unknown length_dist {self.length_dist!r}")
        if self.length_dist == "uniform" and not (0 <= self.min_len <= self.max_len <= self.max_length):
            raise ValueError("degenerate distribution bounds: need 0 <= min_len <= max_len <= max_length")
        if self.length_dist == "lognormal" and self.lognorm_sigma < 0:
            raise ValueError("degenerate distribution bounds: lognorm_sigma must be >= 0")
        if self.embed_dim < 1 or self.num_buckets < 1 or self.max_length < 1:
            raise ValueError("embed_dim, num_buckets and max_length must be >= 1")
        if self.protocol not in PROTOCOLS:
            raise ValueError(f"protocol must be one of {PROTOCOLS}")
        if self.balance_mode not in ("balanced_minichunk", "naive_contiguous"):
            raise ValueError("unknown balance_mode")
        if self.dtype not in DTYPE_SIZES:
            raise ValueError(f"dtype must be one of {sorted(DTYPE_SIZES)}")

    def to_json_dict(self) -> dict:
        """harness.py:97-113 (+ num_heads)."""
        return {
            "cp_size": self.cp_size, "batch_size": self.batch_size, "length_dist": self.length_dist,
            "min_len": self.min_len, "max_len": self.max_len, "lognorm_mu": self.lognorm_mu,
            "lognorm_sigma": self.lognorm_sigma, "max_length": self.max_length, "embed_dim": self.embed_dim,
            "num_buckets": self.num_buckets, "dtype": self.dtype, "protocol": self.protocol,
            "balance_mode": self.balance_mode, "seed": self.seed, "num_heads": self.num_heads,
        }


def draw_lengths(cfg: ExperimentConfig, rng: np.random.Generator) -> np.ndarray:
    """harness.py:116-120."""
    if cfg.length_dist == "uniform":
        return rng.integers(cfg.min_len, cfg.max_len + 1, size=cfg.batch_size)
    raw = np.floor(rng.lognormal(cfg.lognorm_mu, cfg.lognorm_sigma, size=cfg.batch_size))
    return np.clip(raw, 1, cfg.max_length).astype(np.int64)


def gen_synthetic_host(cfg: ExperimentConfig, rank: int) -> dict:
    """harness.py:123-145 on the host: dict of numpy arrays (q/k/v in the drawn dtype)."""
    rng = np.random.default_rng([cfg.seed, rank])
    seq_lengths = draw_lengths(cfg, rng)
    offsets = np.concatenate([[0], np.cumsum(seq_lengths)]).astype(np.int64)
    total = int(offsets[-1])
    # the reference draws in the config's dtype (harness.py:130-133, jagged.py:17);
    # bf16 (this repo's tag) draws the f64 stream and is rounded on the device,
    # so starts / gaps / timestamps are the reference's for the same seed
    dt = np.float32 if cfg.dtype == "f32" else np.float64
    q = rng.standard_normal((total, cfg.embed_dim), dtype=dt)
    k = rng.standard_normal((total, cfg.embed_dim), dtype=dt)
    v = rng.standard_normal((total, cfg.embed_dim), dtype=dt)
    starts = rng.integers(0, 1_000_000_000, size=cfg.batch_size)
    gaps = rng.integers(1, MAX_TS_GAP_SECONDS + 1, size=total)
    ts = np.zeros(total, dtype=np.int64)
    for b in range(cfg.batch_size):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        ts[lo:hi] = starts[b] + np.cumsum(gaps[lo:hi])
    return {"q": q, "k": k, "v": v, "ts": ts, "offsets": offsets}


def gen_synthetic_batch(cfg: ExperimentConfig, rank: int, device=None):
    """harness.py:123-145 -> cp_engine.QKVBatch on the GPU (bf16 values)."""
    from .cp_engine import QKVBatch
    h = gen_synthetic_host(cfg, rank)
    return QKVBatch(
        q=new_jagged(h["q"], h["offsets"], cfg.max_length, device),
        k=new_jagged(h["k"], h["offsets"], cfg.max_length, device),
        v=new_jagged(h["v"], h["offsets"], cfg.max_length, device),
        ts=new_int_series(h["ts"], h["offsets"], device),
    )


def bias_for_config(cfg: ExperimentConfig):
    """harness.py:148-152 (seed + 0x5EED)."""
    bias_cfg = BiasConfig(num_buckets=cfg.num_buckets)
    return BiasParams.normal_init(bias_cfg, seed=cfg.seed + 0x5EED), bias_cfg


def output_errors(got, want) -> tuple[float, float]:
    """harness.py:189-206: (max abs, max row-normalized error)."""
    max_abs = max_rel = 0.0
    for g, w in zip(got, want):
        g = g.values if hasattr(g, "values") else g
        w = w.values if hasattr(w, "values") else w
        g = g.detach().float().cpu().numpy() if isinstance(g, torch.Tensor) else np.asarray(g, np.float64)
        w = w.detach().float().cpu().numpy() if isinstance(w, torch.Tensor) else np.asarray(w, np.float64)
        if g.shape[0] == 0:
            continue
        diff = np.abs(g.astype(np.float64) - w.astype(np.float64))
        ref = np.abs(w.astype(np.float64))
        max_abs = max(max_abs, float(diff.max()))
        max_rel = max(max_rel, float((diff.max(axis=1) / np.maximum(1.0, ref.max(axis=1))).max()))
    return max_abs, max_rel


# --------------------------------------------------------------- experiment

def concat_batches(batches):
    """harness.py:155-170: the CP group's combined batch, sequences in rank order."""
    from .cp_engine import QKVBatch
    offs = [0]
    for b in batches:
        base = offs[-1]
        offs.extend(int(base + o) for o in b.q.host_offsets[1:])
    offs = np.asarray(offs, dtype=np.int64)
    ml = max(b.q.max_length for b in batches)
    cat = lambda f: torch.cat([getattr(b, f).values for b in batches])  # noqa: E731
    return QKVBatch(q=new_jagged(cat("q"), offs, ml, copy=False), k=new_jagged(cat("k"), offs, ml, copy=False),
                    v=new_jagged(cat("v"), offs, ml, copy=False), ts=new_int_series(cat("ts"), offs))


def reference_outputs(batches, params, bias_cfg, num_heads: int = 1):
    """harness.py:173-186: single-device forward over the combined batch (the
    fused kernel), split back per rank."""
    from .attention import AttentionInputs, hstu_attention_reference
    from .jagged import JaggedTensor
    c = concat_batches(batches)
    out = hstu_attention_reference(AttentionInputs(c.q, c.k, c.v, c.ts, params, bias_cfg, num_heads=num_heads))
    res, row = [], 0
    for b in batches:
        n = int(b.q.host_offsets[-1])
        res.append(JaggedTensor(out.values[row:row + n], b.q.offsets, b.q.max_length, b.q.host_offsets))
        row += n
    return res


def redistribution_peaks(batches, cp_size: int, balance_mode: str, protocol: str) -> list:
    """harness.py:256-267: per-rank peak resident bytes of one redistribution protocol."""
    from .comm import RankGroup
    from .cp_engine import build_shard_plan, redistribute_allgather_split, redistribute_alltoall
    from .jagged import lengths
    plan = build_shard_plan([lengths(b.q).tolist() for b in batches], cp_size, balance_mode)
    fn = redistribute_allgather_split if protocol == "allgather_split" else redistribute_alltoall
    _, stats = fn(RankGroup(cp_size), batches, plan)
    return [s.peak_resident_bytes for s in stats]


@dataclass
class ExperimentReport:
    """harness.py:213-253 (same JSON schema; the GPU timing of the pipeline is
    reported under ``metadata.gpu``)."""

    config: ExperimentConfig
    max_abs_error: float
    max_rel_error: float
    redistribute_stats: list
    ring_stats: list
    restore_stats: list
    flops_per_rank: list
    flops_total: int
    flops_max_mean_ratio: float
    resident_tokens_per_rank: list
    per_rank_peak_resident_bytes: list
    redistribute_peak_allgather: list
    redistribute_peak_alltoall: list
    memory_reduction_ratio: float
    gpu: dict

    def to_json_dict(self) -> dict:
        st = lambda xs: [x.to_json_dict() for x in xs]  # noqa: E731
        return {
            "config": self.config.to_json_dict(),
            "max_abs_error": self.max_abs_error,
            "max_rel_error": self.max_rel_error,
            "comm": {"redistribute": st(self.redistribute_stats), "ring": st(self.ring_stats),
                     "restore": st(self.restore_stats)},
            "flops": {"per_rank": self.flops_per_rank, "total": self.flops_total,
                      "max_mean_ratio": self.flops_max_mean_ratio},
            "resident_tokens_per_rank": self.resident_tokens_per_rank,
            "per_rank_peak_resident_bytes": self.per_rank_peak_resident_bytes,
            "redistribute_peak_bytes": {"allgather_split": self.redistribute_peak_allgather,
                                        "alltoall": self.redistribute_peak_alltoall},
            "memory_reduction_ratio": self.memory_reduction_ratio,
            "metadata": {"accounting": ACCOUNTING_NOTE, "gpu": self.gpu},
        }


def run_experiment(cfg: ExperimentConfig, scheduling: str = "sequential", device=None,
                   reference=None) -> ExperimentReport:
    """harness.py:270-316 on the GPU path: the CP pipeline (cp_engine.run_pipeline,
    fused kernels) against a single-device reference, plus both protocols'
    redistribution peaks; ``metadata.gpu`` carries the pipeline's device time
    (CUDA events).  ``reference(batches, params, bias_cfg, num_heads)`` returns
    the per-rank expected outputs; the default is the single-device fused
    forward over the combined batch (as harness.py:173-186 uses its own
    single-device path); tests inject the CPU oracle here."""
    from .cp_engine import run_pipeline
    if scheduling not in SCHEDULINGS:
        raise ValueError(f"unknown scheduling {scheduling!r}")
    batches = [gen_synthetic_batch(cfg, r, device) for r in range(cfg.cp_size)]
    params, bias_cfg = bias_for_config(cfg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    result = run_pipeline(batches, cfg.cp_size, cfg.protocol, cfg.balance_mode, params, bias_cfg, scheduling,
                          num_heads=cfg.num_heads)
    ev[1].record()
    want = (reference or reference_outputs)(batches, params, bias_cfg, cfg.num_heads)
    max_abs, max_rel = output_errors(result.outputs, want)
    if not (np.isfinite(max_abs) and np.isfinite(max_rel)):
        raise RuntimeError(f"non-finite equivalence error: abs={max_abs} rel={max_rel}")
    ag = redistribution_peaks(batches, cfg.cp_size, cfg.balance_mode, "allgather_split")
    a2a = redistribution_peaks(batches, cfg.cp_size, cfg.balance_mode, "alltoall")
    reduction = 1.0 - (max(a2a) / max(ag)) if max(ag) else 0.0
    torch.cuda.synchronize()
    ms = float(ev[0].elapsed_time(ev[1]))
    # attention work of the forward pipeline: 2 GEMMs x 2 d flops per visible (causal) pair per head
    fwd_flops = 4.0 * (cfg.embed_dim // cfg.num_heads) * cfg.num_heads * float(result.flops.total)
    gpu = {"pipeline_ms": ms, "device": torch.cuda.get_device_name(),
           "attention_flops": fwd_flops, "attention_tflops": fwd_flops / max(ms, 1e-9) / 1e9,
           "note": "global-view pipeline (simulated collectives, fused sm_100a kernels); the time includes the "
                   "redistribution / restore row moves and the host-side plan"}
    return ExperimentReport(cfg, max_abs, max_rel, result.redistribute_stats, result.ring_stats,
                            result.restore_stats, list(result.flops.per_rank), result.flops.total,
                            result.flops.max_mean_ratio, list(result.resident_tokens),
                            list(result.peak_resident_bytes), ag, a2a, reduction, gpu)


# ------------------------------------------------------- memory-budget sweep

def modeled_rank_bytes(seq_length: int, cp_size: int, embed_dim: int, dtype_size: int) -> int:
    """harness.py:321-341: modelled per-rank peak for one sequence under the
    balanced shard (q/k/v/ts slabs + output slab + the largest score block)."""
    from .jagged import chunk_assignment, make_minichunks
    sizes = make_minichunks([seq_length], cp_size).chunk_lengths[0]
    t = max(sizes[a] + sizes[b] for a, b in chunk_assignment(cp_size).values())
    largest = max(sizes)
    return t * (3 * embed_dim * dtype_size + 8) + t * embed_dim * dtype_size + t * largest * dtype_size


@dataclass
class SweepReport:
    """harness.py:344-366."""

    budget_bytes: int
    embed_dim: int
    dtype: str
    seed: int
    rows: list
    model: str = ("per-rank token slabs (q/k/v/ts + output) plus largest score block; "
                  "balanced mini-chunk shard of a single sequence")

    def to_json_dict(self) -> dict:
        return {"budget_bytes": self.budget_bytes, "embed_dim": self.embed_dim, "dtype": self.dtype,
                "seed": self.seed, "rows": self.rows, "metadata": {"model": self.model}}


def sweep_max_tokens(budget_bytes: int, cp_sizes, embed_dim: int = 8, dtype: str = "f32", seed: int = 0) -> SweepReport:
    """harness.py:369-394: largest single-sequence length whose modelled per-rank
    footprint fits the budget, per CP size (the model is monotone: doubling,
    then bisection).  ``bench.py`` reports the measured counterpart on the GPU
    (max_seq_len)."""
    if dtype not in DTYPE_SIZES:
        raise ValueError(f"dtype must be one of {sorted(DTYPE_SIZES)}")
    ds = DTYPE_SIZES[dtype]
    rows = []
    for cp in cp_sizes:
        if cp < 1:
            raise ValueError("cp sizes must be >= 1")
        if modeled_rank_bytes(1, cp, embed_dim, ds) > budget_bytes:
            raise ValueError(f"budget {budget_bytes} too small for a single token at cp={cp}")
        lo, hi = 1, 2
        while modeled_rank_bytes(hi, cp, embed_dim, ds) <= budget_bytes:
            lo, hi = hi, hi * 2
            if hi > 1 << 31:
                break
        while lo + 1 < hi:
            mid = (lo + hi) // 2
            if modeled_rank_bytes(mid, cp, embed_dim, ds) <= budget_bytes:
                lo = mid
            else:
                hi = mid
        rows.append({"cp_size": int(cp), "max_supported_length": int(lo)})
    return SweepReport(int(budget_bytes), embed_dim, dtype, seed, rows)


def protocol_memory_measured(lengths, cp_sizes=(2, 4, 8), embed_dim: int = 512, num_heads: int = 4,
                             num_buckets: int = 16, device=None) -> list:
    """MEASURED per-rank transient memory of the batch -> sequence
    redistribution of q, k, v, ts (CPAttention.redistribute) under the two
    protocols -- the measured counterpart of ``redistribution_peaks``
    (harness.py:256-267; the paper's -60 % for all-to-all).
    Every rank holds ``lengths`` (cp_layer.LoopbackComm: one rank's buffers,
    communication excluded).  Rows: cp, peak bytes above the inputs for
    "alltoall" and "allgather_split", and their ratio."""
    from .cp_layer import CPAttention, LoopbackComm
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    lens = np.asarray(lengths, dtype=np.int64)
    T = int(lens.sum())
    gen = torch.Generator(device=dev).manual_seed(3)
    q, k, v = (torch.randn(T, embed_dim, device=dev, generator=gen).bfloat16() for _ in range(3))
    ts = torch.cumsum(torch.randint(1, 10**6, (T,), device=dev, generator=gen), 0)
    rows = []
    for cp_size in cp_sizes:
        row = {"cp_size": int(cp_size)}
        for protocol in ("alltoall", "allgather_split"):
            cp = CPAttention(None, num_heads, num_buckets, comm=LoopbackComm(cp_size, 0), protocol=protocol)
            plan = cp.plan_for(lens, dev)
            torch.cuda.synchronize(dev)
            torch.cuda.empty_cache()
            torch.cuda.reset_peak_memory_stats(dev)
            base = torch.cuda.memory_allocated(dev)
            res = [cp.redistribute(x, *plan) for x in (q, k, v)] + [cp.redistribute(ts.view(-1, 1), *plan)]
            torch.cuda.synchronize(dev)
            row[f"{protocol}_peak_bytes"] = int(torch.cuda.max_memory_allocated(dev) - base)
            row[f"{protocol}_resident_rows"] = int(res[0].shape[0])
            del res, cp, plan
        row["allgather_split_over_alltoall"] = round(row["allgather_split_peak_bytes"] /
                                                     max(row["alltoall_peak_bytes"], 1), 2)
        rows.append(row)
    return rows


def sweep_max_tokens_measured(budget_bytes: int, cp_sizes=(1, 2, 4, 8), embed_dim: int = 512, num_heads: int = 4,
                              num_layers: int = 8, num_buckets: int = 16, seed: int = 7, granularity: int = 2048,
                              time_budget_s: float = 200.0, device=None, rel_precision: float = 1 / 128) -> SweepReport:
    """The MEASURED counterpart of ``sweep_max_tokens`` (harness.py:369-394) on
    the GPU: for each CP size, the longest single sequence whose per-rank share
    -- its two balanced mini-chunks through ``num_layers`` HSTU layers, K/V of
    the whole sequence gathered per layer and re-gathered in the backward --
    runs forward + backward under a per-process memory cap of ``budget_bytes``
    (torch.cuda.set_per_process_memory_fraction).  Communication is excluded
    (cp_layer.LoopbackComm: one rank's memory and kernel work, the peers' K/V
    replaced by replicas).  Doubling (from 8 * granularity, or from the
    previous CP size's maximum: it can only grow with CP), then bisection to
    ``granularity`` tokens or ``rel_precision`` of the length, whichever is
    coarser (granularity: a multiple of 2 * cp * 128 for every cp <= 8).
    Rows carry ``max_supported_length`` (the reference's key), the first
    failing length, the peak allocated bytes at the maximum and the ratio to
    the first CP size."""
    import time

    from .cp_layer import CPAttention, LoopbackComm
    from .hstu_layer import HSTUStack
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if embed_dim % num_heads:
        raise ValueError("embed_dim must be divisible by num_heads")
    head_dim = embed_dim // num_heads
    total = torch.cuda.get_device_properties(dev).total_memory
    if budget_bytes <= 0 or budget_bytes > total:
        raise ValueError(f"budget {budget_bytes} must be in (0, {total}] bytes")
    from . import kernels
    kernels.release_caches()
    torch.cuda.empty_cache()
    torch.cuda.set_per_process_memory_fraction(budget_bytes / total, dev)
    t0 = time.time()

    def runs(k: int, L: int):
        try:
            comm = LoopbackComm(k, 0, peer_lengths=lambda r: [])
            cp = CPAttention(None, num_heads, num_buckets, comm=comm)
            st = HSTUStack(num_layers, embed_dim, num_heads, head_dim, num_buckets, seed=seed, cp=cp).to(dev)
            plan = cp.plan_for([L], dev)
            n = plan[0].n_res
            gen = torch.Generator(device=dev).manual_seed(L)
            x = torch.randn(n, embed_dim, device=dev, generator=gen).bfloat16().requires_grad_(True)
            ts = torch.cumsum(torch.randint(1, 10**6, (n,), device=dev, generator=gen), 0)
            y = x
            for layer in st.layers:
                y = layer(y, ts, cp=(cp, plan))
            y.float().sum().backward()
            torch.cuda.synchronize()
            peak = torch.cuda.max_memory_allocated(dev)
            del st, x, y
            ok = True
        except torch.OutOfMemoryError:
            ok, peak = False, None
        except RuntimeError as e:
            if "out of memory" not in str(e).lower():
                raise
            ok, peak = False, None
        kernels.release_caches()
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(dev)
        return ok, peak

    rows = []
    try:
        for k in cp_sizes:
            if k < 1:
                raise ValueError("cp sizes must be >= 1")
            lo, hi, peak_lo, L = 0, None, None, 8 * granularity
            if rows and rows[-1]["max_supported_length"] >= L:  # start from the previous CP size's maximum
                L = rows[-1]["max_supported_length"]
            while hi is None and time.time() - t0 < time_budget_s:
                ok, pk = runs(k, L)
                if ok:
                    lo, peak_lo, L = L, pk, 2 * L
                else:
                    hi = L
            while (hi is not None and hi - lo > max(granularity, int(lo * rel_precision))
                   and time.time() - t0 < time_budget_s):
                mid = (lo + hi) // 2 // granularity * granularity
                ok, pk = runs(k, mid)
                if ok:
                    lo, peak_lo = mid, pk
                else:
                    hi = mid
            rows.append({"cp_size": int(k), "max_supported_length": int(lo), "first_failure": hi,
                         "peak_gb_at_max": None if peak_lo is None else round(peak_lo / 1e9, 2)})
    finally:
        torch.cuda.set_per_process_memory_fraction(1.0, dev)
    base = rows[0]["max_supported_length"] if rows and rows[0]["max_supported_length"] else None
    for r in rows:
        r["vs_first"] = None if not base else round(r["max_supported_length"] / base, 2)
    model = (f"measured on {torch.cuda.get_device_name(dev)}: one rank's share of one sequence through "
             f"{num_layers} HSTU layers (E={embed_dim}, H={num_heads}), fwd+bwd under a per-process memory cap; "
             f"communication excluded (LoopbackComm); granularity {granularity}; {round(time.time() - t0, 1)} s")
    return SweepReport(int(budget_bytes), embed_dim, "bf16", seed, rows, model)
