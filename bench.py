#!/usr/bin/env python
"""Benchmark: jagged HSTU attention fwd+bwd tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1  -> config C2 (BASELINE.json configs[1]): B=32 sequences, lengths
          uniform[1,1024], H=4 heads, d=128, bf16, reference generator seed 7.
N > 1  -> jagged context parallelism over N ranks (one process per GPU,
          torchrun, NCCL): each rank contributes B=32 sequences (per-rank batch
          fixed -> weak scaling), sharded by the balanced 2*CP mini-chunk plan.

A step is one forward + backward of the attention over the whole batch.
``value`` = tokens of all ranks / device step time (inputs resident, L2
flushed between timed steps); ``e2e`` = the same through the public API with
host (pinned) inputs copied H2D and every result (out, dq, dk, dv,
d_ts_weights) read back D2H inside the timed region.  ``--impl reference``
times the reference's own CPU path (jaggedcp installed in baseline/_ref,
through its public API) on host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HSTU jagged attn fwd+bwd tokens/sec"
UNIT = "tokens/s"
SEED = 7
B, MAXLEN, H, D = 32, 1024, 4, 128
NB = 16


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), float(
            p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def _host_batch(rank: int):
    from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host
    cfg = ExperimentConfig(cp_size=1, batch_size=B, min_len=1, max_len=MAXLEN, max_length=MAXLEN,
                           embed_dim=H * D, seed=SEED)
    return gen_synthetic_host(cfg, rank)


def _ts_weights():
    from paper_2508_04711_b200.attention import BiasConfig, BiasParams
    return BiasParams.normal_init(BiasConfig(NB), SEED + 0x5EED).ts_weights


def _flops(lengths) -> float:
    s = float(sum(int(L) * (int(L) + 1) for L in lengths))
    return 7.0 * D * H * s, 2.0 * D * H * s, 5.0 * D * H * s


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region
    (NVML every ~1 ms in a thread; nvidia-smi -lms as a fallback)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.rows = []
        self.thread = None

    def _nvml_loop(self, nv, handle):
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        mx = nv.nvmlDeviceGetMaxClockInfo(handle, nv.NVML_CLOCK_SM)
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(handle)
                self.rows.append((float(sm), float(mx), ["Active" if rs & b else "Not Active" for b in bits]))
            except Exception:
                pass
            self.ready.set()
            time.sleep(0.001)

    def __enter__(self):
        self.stop = False
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            handle = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.ready = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, handle), daemon=True)
            self.thread.start()
            self.ready.wait(2.0)  # the timed region is a few ms: be sampling before it starts
        except Exception:
            self.thread = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                     "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.proc = None
            time.sleep(0.5)
        return self

    def __exit__(self, *a):
        self.stop = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for line in (out or "").strip().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 6:
                    try:
                        self.rows.append((float(parts[0]), float(parts[1]), parts[2:6]))
                    except ValueError:
                        pass

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({self.NAMES[i] for _, _, flags in rows for i, f in enumerate(flags)
                          if f.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


# --------------------------------------------------------------------- GPU arm

def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # JH_BENCH_TEST_GLOO=1 (tests only): N > 1 ranks on ONE GPU, exchanging over gloo
    # through host memory (cp_layer.HostStagedComm) -- exercises this script's
    # multi-rank logic where only one GPU exists; never a measurement
    test_gloo = world > 1 and os.environ.get("JH_BENCH_TEST_GLOO") == "1"
    if test_gloo:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if test_gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def allreduce_max(x: float) -> float:
        t = torch.tensor([x], device="cpu" if test_gloo else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_2508_04711_b200 import kernels
    from paper_2508_04711_b200.attention import (AttentionInputs, BiasConfig, BiasParams,
                                                 hstu_attention_backward, hstu_attention_reference)
    from paper_2508_04711_b200.jagged import new_int_series, new_jagged

    h = _host_batch(rank)
    lens = np.diff(h["offsets"])
    T = int(h["offsets"][-1])
    rng = np.random.default_rng([SEED, 99, rank])
    g_host = rng.standard_normal((T, H * D), dtype=np.float32)
    w_host = _ts_weights()

    q = torch.from_numpy(h["q"]).to(dev).bfloat16()
    k = torch.from_numpy(h["k"]).to(dev).bfloat16()
    v = torch.from_numpy(h["v"]).to(dev).bfloat16()
    g = torch.from_numpy(g_host).to(dev).bfloat16()
    ts = torch.from_numpy(h["ts"]).to(dev)
    offs = torch.from_numpy(h["offsets"]).to(dev)
    w = torch.from_numpy(w_host.astype(np.float32)).to(dev)

    cp_size = world if args.cp <= 0 else args.cp
    if world > 1:
        from paper_2508_04711_b200.cp_layer import CPAttention, make_cp_dp_groups
        if cp_size == world:
            cp_group, dp_group = dist.group.WORLD, None
        else:  # hybrid CP x DP (config C5): CP groups of consecutive ranks, DP across them
            cp_group, dp_group, _, _ = make_cp_dp_groups(cp_size)
        if test_gloo:
            from paper_2508_04711_b200.cp_layer import HostStagedComm
            cp = CPAttention(cp_group, H, NB, protocol=args.protocol, comm=HostStagedComm(cp_group))
        else:
            cp = CPAttention(cp_group, H, NB, protocol=args.protocol)
        cp_step = cp.bench_step(q, k, v, ts, h["offsets"], g, w)

        def step_fn(prof=None):
            dq_, dk_, dv_, dw_ = cp_step()
            if dp_group is not None:  # DDP rule: summed over CP (inside), averaged over DP
                if test_gloo:
                    h_ = dw_.cpu()
                    dist.all_reduce(h_, group=dp_group)
                    dw_.copy_(h_)
                else:
                    dist.all_reduce(dw_, group=dp_group)
                dw_ /= world // cp_size
            return dq_, dk_, dv_, dw_
        all_lens = [None] * world
        dist.all_gather_object(all_lens, [int(x) for x in lens])
        tokens_total = sum(sum(x) for x in all_lens)
        flat_lens = [x for r in all_lens for x in r]
    else:
        band = kernels.new_band_table(T, len(lens), dev)  # computed by the forward, reused by the backward
        seg_host = (h["offsets"], None, None)
        bwd_two_kernel = kernels.ds_scratch_bytes(H, h["offsets"]) <= kernels.ds_scratch_budget(dev)

        def step_fn(prof=None):
            if prof is None:  # forward and backward concurrently on two streams (kernels.attn_fwd_bwd)
                return kernels.attn_fwd_bwd(q, k, v, ts, offs, g, H, w, NB, seg_host=seg_host, band_table=band)[1:]
            # the per-kernel (roofline) pass: the two calls in sequence, CUDA events around each kernel
            kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, NB, prof=prof[0], band_table=band)
            return kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, NB, prof=prof[1], seg_host=seg_host,
                                    band_table=band)
        tokens_total = T
        flat_lens = [int(x) for x in lens]

    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_fn()
    barrier()

    # N = 1: the step (work-list builds + 3 attention kernels + d_w zeroing) is
    # captured once into a CUDA graph and replayed, so host launch overhead is
    # not on the device timeline.  The per-kernel roofline timing below uses a
    # separate eager pass with events around the kernels.
    graph = None
    if world == 1 and not args.no_graph:
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for _ in range(2):
                step_fn()
        stream.wait_stream(side)
        barrier()
        graph = torch.cuda.CUDAGraph()
        n0 = kernels.launch_count()
        with torch.cuda.graph(graph):
            step_fn()
        launches_per_step = kernels.launch_count() - n0
        barrier()
        graph.replay()
        barrier()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    kev = [((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)),
            (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))) for _ in range(K)]
    launches0 = kernels.launch_count()
    with Clocks(local) as clk:
        barrier()
        for i in range(K):
            flush.fill_(float(i))  # evict the step's inputs from L2 (512 MiB > 126 MB L2)
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step_fn(prof=kev[i] if world == 1 else None)
            ev[i][1].record(stream)
        barrier()
    launches = (kernels.launch_count() - launches0) if graph is None else launches_per_step * K
    if graph is not None:
        # eager pass for the per-kernel (roofline) timings
        for i in range(K):
            flush.fill_(float(i))
            step_fn(prof=kev[i])
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    if world > 1:
        total_ms = allreduce_max(total_ms)
    ms_per_step = total_ms / K
    value = tokens_total / (ms_per_step / 1e3)

    peak, peak_sus, hbm, peak_kind = _peaks()
    F, Ff, Fb = _flops(flat_lens)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (reference generator harness.py:123, seed 7; q/k/v/dO bf16)",
        "config": {"workload": "C2: jagged HSTU attention fwd+bwd, B=32/rank, lengths uniform[1,1024], "
                               "H=4, d=128, nb=16" + ("" if world == 1 else f", jagged CP={world} (balanced)"),
                   "batch_per_rank": B, "max_seq_len": MAXLEN, "heads": H, "head_dim": D, "tokens": tokens_total,
                   "parallelism": "single" if world == 1 else (f"cp{world}" if cp_size == world
                                                                else f"cp{cp_size}xdp{world // cp_size}"),
                   "cp_protocol": None if world == 1 else args.protocol,
                   "l2": "flushed between timed steps (512 MiB write, outside the timed events)",
                   "cuda_graph": graph is not None,
                   "schedule": ("band table, then forward || backward on two streams (kernels.attn_fwd_bwd; the HSTU "
                                "backward recomputes from q, k, v)") if world == 1 else "CP layer forward, backward"},
        "tflops": F / (ms_per_step / 1e3) / 1e12,
        "tensor_frac_step": F / (ms_per_step / 1e3) / (world * peak * 1e12),
        "gpu_launches": int(launches),
    }
    if world == 1:
        fwd_ms = float(np.mean([a.elapsed_time(b) for (a, b), _ in kev]))
        bwd_ms = float(np.mean([a.elapsed_time(b) for _, (a, b) in kev]))
        ach_b = Fb / (bwd_ms / 1e3) / 1e12
        ach_f = Ff / (fwd_ms / 1e3) / 1e12
        result["roofline"] = {
            "bound": "tensor",
            "kernel": ("jh_attn_bwd: hstu_bwd_dkv_kernel<128> + hstu_bwd_dq_kernel<128>" if bwd_two_kernel
                       else "jh_attn_bwd: hstu_bwd_fused_kernel<128>"), "achieved": ach_b, "peak": peak,
            "unit": "TFLOP/s", "frac": ach_b / peak, "traffic": _traffic("bwd"),
            "peak_kind": f"{peak_kind} burst bf16 (MEASURED_PEAKS.json)",
            "algorithmic_flops_per_launch": Fb, "ms_per_launch": bwd_ms,
            "fwd": {"kernel": "hstu_fwd2_kernel<128>" if os.environ.get("JH_FWD2") == "1" else "hstu_fwd_kernel<128>", "achieved": ach_f, "frac": ach_f / peak,
                    "algorithmic_flops_per_launch": Ff, "ms_per_launch": fwd_ms, "traffic": _traffic("fwd")},
        }
    result["clocks"] = clk.summary()
    if test_gloo:
        result["test_mode"] = "JH_BENCH_TEST_GLOO: all ranks on cuda:0, gloo host-staged exchange -- not a measurement"

    # ---------------- e2e through the public API with host buffers
    import torch as _t
    pin = lambda a: _t.from_numpy(a).pin_memory()  # noqa: E731
    qh, kh, vh = (pin(h[x]).bfloat16().pin_memory() for x in ("q", "k", "v"))
    gh = pin(g_host).bfloat16().pin_memory()
    tsh, offh = pin(h["ts"]), h["offsets"]
    params, bcfg = BiasParams(w_host), BiasConfig(NB)
    h2d = sum(x.numel() * x.element_size() for x in (qh, kh, vh, gh, tsh)) + 5 * offh.nbytes + 2 * NB * 4
    # results back to pinned host buffers: out, dq, dk, dv (bf16) and d_ts_weights (f64),
    # i.e. everything the reference's numpy API returns
    outs_h = [torch.empty((T, H * D), dtype=torch.bfloat16).pin_memory() for _ in range(4)]
    dw_h = torch.empty(NB, dtype=torch.float64).pin_memory()
    d2h_full = sum(x.numel() * x.element_size() for x in outs_h) + dw_h.numel() * 8
    d2h_dw = NB * 8

    def e2e_step(full: bool):
        qj = new_jagged(qh.to(dev, non_blocking=True), offh, MAXLEN, copy=False)
        kj = new_jagged(kh.to(dev, non_blocking=True), offh, MAXLEN, copy=False)
        vj = new_jagged(vh.to(dev, non_blocking=True), offh, MAXLEN, copy=False)
        tj = new_int_series(tsh.to(dev, non_blocking=True), offh)
        inp = AttentionInputs(qj, kj, vj, tj, params, bcfg, num_heads=H)
        out = hstu_attention_reference(inp)
        gr = hstu_attention_backward(inp, new_jagged(gh.to(dev, non_blocking=True), offh, MAXLEN, copy=False))
        if full:
            for dst, src in zip(outs_h, (out.values, gr.dq.values, gr.dk.values, gr.dv.values)):
                dst.copy_(src, non_blocking=True)
        dw_h.copy_(gr.d_ts_weights, non_blocking=True)

    def e2e_time(full: bool):
        for _ in range(max(args.warmup, 3)):
            e2e_step(full)
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(K):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step(full)
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / K

    from paper_2508_04711_b200.attention import hstu_attention_fwd_bwd_host, hstu_attention_fwd_bwd_host_async
    pipe_info = {}
    outs_h2 = [torch.empty((T, H * D), dtype=torch.bfloat16).pin_memory() for _ in range(4)]

    def pipe_time():
        """Back-to-back steps through the async host-streaming call: step i+1's
        inputs copy in while step i's results copy out (two output buffer sets,
        step i waited for before its buffers are reused).  Every step still
        moves all of its inputs H2D and all of its results D2H."""
        sets = (outs_h, outs_h2)

        def run(n):  # n calls, two in flight
            prev = None
            for i in range(n):
                cur = hstu_attention_fwd_bwd_host_async(qh, kh, vh, tsh, offh, gh, w_host, H, NB,
                                                        groups=args.e2e_groups, out=sets[i % 2])
                if prev is not None:
                    prev.wait()
                prev = cur
            prev.wait()

        # warm-up in the same two-in-flight pattern, long enough for the caching
        # allocators to hold every buffer of two calls in flight (the first ~8
        # calls of a process allocate: scripts/e2e_pipe_probe.py)
        run(max(args.warmup, 3) + 9)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        run(K)
        wall = time.perf_counter() - t0
        e1.record(stream)
        e1.synchronize()
        pipe_info["wall_ms_per_step"] = wall / K * 1e3
        return e0.elapsed_time(e1) / K

    def stream_step():
        return hstu_attention_fwd_bwd_host(qh, kh, vh, tsh, offh, gh, w_host, H, NB, groups=args.e2e_groups,
                                           out=outs_h)

    def stream_time():
        for _ in range(max(args.warmup, 3)):
            stream_step()
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(K):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            stream_step()  # returns after the last result reached the host
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / K

    if world == 1 and not args.no_e2e:
        e2e_ms = pipe_time()
        call_ms = stream_time()
        api_ms = e2e_time(True)
        e2e_dw_ms = e2e_time(False)
        result["e2e"] = {"value": T / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                         "d2h_bytes_per_step": int(d2h_full), "ms_per_step": e2e_ms,
                         "returns": "out, dq, dk, dv (bf16) + d_ts_weights (f64) in host memory",
                         "api": "paper_2508_04711_b200.attention.hstu_attention_fwd_bwd_host_async, steps back to "
                                "back (step i+1's inputs copy in while step i's results copy out; "
                                f"{args.e2e_groups} sequence runs per step over copy / compute streams); inputs "
                                "arrive over PCIe every step, so no L2 flush",
                         "wall_ms_per_step": pipe_info.get("wall_ms_per_step"),
                         "per_call": {"value": T / (call_ms / 1e3), "ms_per_step": call_ms,
                                      "api": "hstu_attention_fwd_bwd_host (synchronous: each call returns with its "
                                             "results on the host; L2 flushed between calls)"},
                         "jagged_api": {"value": T / (api_ms / 1e3), "ms_per_step": api_ms,
                                        "api": "hstu_attention_reference + hstu_attention_backward on JaggedTensors, "
                                               "copies before / after (not overlapped)"},
                         "d_ts_weights_only": {"value": T / (e2e_dw_ms / 1e3), "d2h_bytes_per_step": int(d2h_dw),
                                               "ms_per_step": e2e_dw_ms}}
    else:
        result["e2e"] = None

    if world > 1:
        # one extra, untimed step with CUDA events around every collective: bytes,
        # GB/s against NVLink 5 and the exposed (non-overlapped) exchange time
        cp.meter = {"coll": [], "join": []}
        step_fn()
        rep = cp.exchange_report()
        rep["exposed_ms_max_over_ranks"] = allreduce_max(rep.get("exposed_ms", 0.0))
        result["cp_exchange"] = rep
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(h, g_host, w_host)
    if world == 1 and not args.no_stack:
        result["stack"] = stack_bench(dev, max(3, min(K, 10)), flush)
    if world == 1 and not args.no_max_len:
        del flush
        torch.cuda.empty_cache()
        result["max_seq_len"] = max_seq_len_probe(dev, w)
    if world == 1:
        from paper_2508_04711_b200.harness import protocol_memory_measured
        lens4, _ = _c4_batch()
        result["protocol_memory"] = {
            "workload": "C4 per-rank batch (rank 0's 4 sequences, lognormal(ln 1024, 1.0), E=512) on every rank: "
                        "per-rank transient bytes of redistributing q, k, v, ts (communication excluded, "
                        "LoopbackComm)",
            "rows": protocol_memory_measured(lens4[:4], (2, 4, 8), embed_dim=C4_E, num_heads=H, device=dev)}
    if world == 1 and args.cp_sweep_gb > 0:
        result["cp_sweep"] = cp_sweep(dev, args.cp_sweep_gb)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


C4_E, C4_LAYERS = H * D, 8


def _c4_batch():
    """C4 lengths: 32 sequences, lognormal(ln 1024, 1.0) clipped
    to [1, 8192], reference generator, seed 7 (all CP ranks' batches = rank 0..7
    of the reference convention, B=4 each)."""
    from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host
    parts = []
    for r in range(8):
        cfg = ExperimentConfig(cp_size=8, batch_size=4, length_dist="lognormal", lognorm_mu=float(np.log(1024)),
                               lognorm_sigma=1.0, max_length=8192, embed_dim=8, seed=SEED)
        parts.append(gen_synthetic_host(cfg, r))
    lens = np.concatenate([np.diff(p["offsets"]) for p in parts])
    ts = np.concatenate([p["ts"] for p in parts])
    return lens, ts


def stack_bench(dev, steps: int, flush):
    """8-layer HSTU stack (hstu_layer.HSTUStack, E = H*d = 512) fwd+bwd over the
    whole C4 batch on ONE GPU (CP = 1): tokens/s of the full model step
    (attention kernels + norm_gate / SiLU kernels + cuBLAS GEMMs)."""
    import torch
    from paper_2508_04711_b200 import kernels
    from paper_2508_04711_b200.hstu_layer import HSTUStack
    lens, ts_h = _c4_batch()
    offs_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs_h[-1])
    st = HSTUStack(C4_LAYERS, C4_E, H, D, NB, seed=SEED).to(dev)
    gen = torch.Generator(device=dev).manual_seed(SEED)
    x = torch.randn(T, C4_E, device=dev, generator=gen).bfloat16().requires_grad_(True)
    gy = torch.randn(T, C4_E, device=dev, generator=gen).bfloat16()
    ts, offs = torch.from_numpy(ts_h).to(dev), torch.from_numpy(offs_h).to(dev)
    maxlen = int(lens.max())

    def step():
        x.grad = None
        st.zero_grad(set_to_none=True)
        st(x, ts, offs, maxlen).backward(gy)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    tot = 0.0
    n0 = kernels.launch_count()
    for i in range(steps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / steps
    s2 = float((lens * (lens + 1)).sum())
    f_attn = 7.0 * D * H * s2 * C4_LAYERS
    f_gemm = 6.0 * T * (4 * H * D * C4_E + H * D * C4_E) * C4_LAYERS  # fwd + 2 bwd GEMMs per projection
    return {"workload": f"C4 batch on 1 GPU (CP=1): {C4_LAYERS} HSTU layers, E={C4_E}, H={H}, d={D}, "
                        f"32 sequences lognormal(ln 1024, 1.0) clipped [1, 8192], T={T}",
            "value": T / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "tflops": (f_attn + f_gemm) / (ms / 1e3) / 1e12, "attention_flops": f_attn, "gemm_flops": f_gemm,
            "jh_launches_per_step": (kernels.launch_count() - n0) / steps}


def cp_sweep(dev, cap_gb: float):
    """Measured max supported single-sequence length per CP size under a
    fixed per-GPU memory cap (harness.sweep_max_tokens_measured: one rank's
    share through the 8-layer stack, communication excluded) -- the measured
    analogue of the reference's modeled sweep (harness.py:308-374); the
    paper's claim is 5.3x at CP=8."""
    from paper_2508_04711_b200.harness import sweep_max_tokens_measured
    rep = sweep_max_tokens_measured(int(cap_gb * 1e9), (1, 2, 4, 8), embed_dim=C4_E, num_heads=H,
                                    num_layers=C4_LAYERS, num_buckets=NB, seed=SEED, device=dev)
    rows = [dict(r, vs_cp1=r.pop("vs_first")) for r in rep.rows]
    return {"cap_gb": cap_gb, "layers": C4_LAYERS, "embed_dim": C4_E, "heads": H, "head_dim": D,
            "granularity": 2048, "communication": "excluded (LoopbackComm: one rank's memory and kernel work)",
            "rows": rows, "model": rep.model}


def max_seq_len_probe(dev, w):
    """Longest single sequence (B=1, H=4, d=128, bf16) whose fwd+bwd runs on
    this GPU (the metric's "max supported seq len" at CP=1): lengths double
    from 16K until the first out-of-memory, then a bisection to 4K granularity.
    Each probe is a real fwd+bwd through the kernels on synthetic data (once
    the whole-sequence dS scratch would exceed its budget, the backward's auto
    policy runs kv windows with a bounded scratch, kernels._attn_bwd_windowed)."""
    import torch
    from paper_2508_04711_b200 import kernels

    def runs(L):
        try:
            gen = torch.Generator(device=dev).manual_seed(L)
            q, k, v, g = (torch.randn(L, H * D, device=dev, generator=gen).bfloat16() for _ in range(4))
            ts = torch.cumsum(torch.randint(1, 10**6, (L,), device=dev, generator=gen), 0)
            offs = torch.tensor([0, L], dtype=torch.int64, device=dev)
            kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, NB)
            kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, NB, seg_host=(np.array([0, L]), None, None))
            torch.cuda.synchronize()
            ok = True
        except torch.OutOfMemoryError:
            ok = False
        except RuntimeError as e:  # allocation failures surfaced by the extension
            if "out of memory" not in str(e).lower():
                raise
            ok = False
        torch.cuda.empty_cache()
        return ok

    t0 = time.time()
    lo, hi, L = 0, None, 16384
    while hi is None and L <= (1 << 21) and time.time() - t0 < 90:
        if runs(L):
            lo, L = L, 2 * L
        else:
            hi = L
    if hi is not None:
        while hi - lo > 4096:
            mid = (lo + hi) // 2 // 4096 * 4096
            if runs(mid):
                lo = mid
            else:
                hi = mid
    kernels.release_caches()
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info(dev)
    return {"value": lo, "unit": "tokens", "cp": 1, "batch": 1, "heads": H, "head_dim": D,
            "first_failure": hi, "gpu_memory_gb": round(total / 1e9, 1), "granularity": 4096,
            "binding_term": ("none reached: every buffer is O(L) plus a bounded dS scratch (beyond its "
                             "budget the backward runs kv windows); probe capped at 2^21 tokens / 90 s"),
            "probe_s": round(time.time() - t0, 1)}


def _traffic(which: str):
    """DRAM bytes per launch from the committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(which)
    except Exception:
        return None


# --------------------------------------------------------------------- CPU legs

def _cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = max((i.get("num_threads", 1) for i in info), default=1)
        return int(n), [{k: i.get(k) for k in ("internal_api", "num_threads")} for i in info]
    except Exception:
        return os.cpu_count() or 1, []


def _load_reference():
    """The unmodified reference package installed in baseline/_ref (pip --target,
    DESIGN.md (d)); None when it is absent (then the oracle port stands in)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "jaggedcp")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import jaggedcp
        return jaggedcp
    except Exception:
        return None


def _cpu_fwd_bwd(h, g, w, seq_ids, ref):
    """fwd+bwd of the given sequences, all heads, f32, on the host: through the
    reference's own public API (jaggedcp.hstu_attention_reference /
    hstu_attention_backward, one call per head: the reference is single-head)
    or the oracle port.  Returns (seconds, tokens)."""
    offs = h["offsets"]
    rows = np.concatenate([np.arange(offs[b], offs[b + 1]) for b in seq_ids]) if len(seq_ids) else np.zeros(0, int)
    sub_offs = np.concatenate([[0], np.cumsum([offs[b + 1] - offs[b] for b in seq_ids])]).astype(np.int64)
    bf = lambda a: a[rows].astype(np.float32)  # noqa: E731
    q, k, v, gg = bf(h["q"]), bf(h["k"]), bf(h["v"]), bf(g)
    ts = h["ts"][rows]
    t0 = time.perf_counter()
    if ref is None:
        import oracle
        oracle.hstu_forward(q, k, v, ts, sub_offs, w, NB, H)
        oracle.hstu_backward(q, k, v, ts, sub_offs, gg, w, NB, H)
    else:
        params, cfg = ref.BiasParams(np.asarray(w, dtype=np.float64)), ref.BiasConfig(NB)
        tsj = ref.new_int_series(ts, sub_offs)
        for hh in range(H):
            sl = slice(hh * D, (hh + 1) * D)
            inp = ref.AttentionInputs(ref.new_jagged(q[:, sl], sub_offs, MAXLEN), ref.new_jagged(k[:, sl], sub_offs, MAXLEN),
                                      ref.new_jagged(v[:, sl], sub_offs, MAXLEN), tsj, params, cfg)
            ref.hstu_attention_reference(inp)
            ref.hstu_attention_backward(inp, ref.new_jagged(gg[:, sl], sub_offs, MAXLEN))
    return time.perf_counter() - t0, int(sub_offs[-1])


def cpu_baseline(h, g, w):
    """The reference (baseline/_ref jaggedcp, else the oracle port) on the
    host's cores: the full C2 batch, fwd+bwd, f32, one pass (reported only)."""
    ref = _load_reference()
    cores, info = _cpu_threads()
    secs, toks = _cpu_fwd_bwd(h, g, w, list(range(len(h["offsets"]) - 1)), ref)
    return {"value": toks / secs, "unit": UNIT, "cores": cores, "kind": "port" if ref is None else "reference",
            "sample": f"full C2 batch ({toks} tokens, 32 sequences, 4 heads), fwd+bwd f32, one pass, "
                      f"{secs:.2f} s" + ("" if ref is None else ", jaggedcp from baseline/_ref"),
            "host_cpus": os.cpu_count(), "blas": info}


def run_reference(args):
    """--impl reference: the reference's own CPU path (jaggedcp from
    baseline/_ref through its public API; the oracle port if it is absent) on
    the host cores.  Each step is a bounded sample of the C2 batch: 4
    sequences, taken round-robin so that consecutive steps cycle through the
    whole batch (every 8 steps cover all 32 sequences once)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    ref = _load_reference()
    h = _host_batch(0)
    T = int(h["offsets"][-1])
    rng = np.random.default_rng([SEED, 99, 0])
    g = rng.standard_normal((T, H * D), dtype=np.float32)
    w = _ts_weights()
    nseq = len(h["offsets"]) - 1
    per = 4
    for i in range(args.warmup):
        _cpu_fwd_bwd(h, g, w, [(per * i + j) % nseq for j in range(per)], ref)
    tot_s, tot_tok = 0.0, 0
    for i in range(args.steps):
        s, t = _cpu_fwd_bwd(h, g, w, [(per * i + j) % nseq for j in range(per)], ref)
        tot_s += s
        tot_tok += t
    value = tot_tok / tot_s
    cores, info = _cpu_threads()
    kind = "port" if ref is None else "reference"
    desc = (f"{per} of the 32 C2 sequences per step, round-robin over the batch ({args.steps} steps, "
            f"{tot_tok} tokens), 4 heads, fwd+bwd f32, "
            + ("oracle port (baseline/_ref absent)" if ref is None else
               "unmodified jaggedcp (baseline/_ref) hstu_attention_reference + hstu_attention_backward per head"))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generator harness.py:123, seed 7)",
        "config": {"workload": "C2: jagged HSTU attention fwd+bwd, B=32, lengths uniform[1,1024], H=4, d=128",
                   "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc, "blas": info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a captured CUDA graph")
    ap.add_argument("--no-max-len", action="store_true", help="skip the max-supported-sequence-length probe")
    ap.add_argument("--cp", type=int, default=0, help="CP group size for N > 1 (default: all ranks; "
                    "smaller = hybrid CP x DP)")
    ap.add_argument("--protocol", choices=["alltoall", "allgather_split"], default="alltoall",
                    help="batch -> sequence redistribution protocol for N > 1")
    ap.add_argument("--e2e-groups", type=int, default=2, help="sequence runs of the host-streaming e2e call")
    ap.add_argument("--no-stack", action="store_true", help="skip the 8-layer HSTU stack (C4 batch) measurement")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e legs (profiling runs)")
    ap.add_argument("--cp-sweep-gb", type=float, default=24.0,
                    help="per-GPU memory cap of the CP max-length sweep (0 = skip)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
