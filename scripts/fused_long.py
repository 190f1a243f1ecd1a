"""Long-sequence backward: the fused one-kernel path (O(L) memory) against the
two-kernel path (bf16 dS scratch) where the scratch still fits, and the
windowed two-kernel path (auto mode: JH_WIN_BUDGET bytes of dS scratch, default the
kernels.ds_scratch_budget, 1/8 of the GPU).  Prints time, TF/s and the extra peak memory of each.
--once: one fused call (ncu capture)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402

H, D = 4, 128
dev = "cuda"


def case(L, B):
    torch.manual_seed(L)
    T = L * B
    q, k, v, g = (torch.randn(T, H * D, device=dev).bfloat16() for _ in range(4))
    ts = torch.cumsum(torch.randint(100_000, 1_000_000, (T,), device=dev), 0)
    offs_h = np.arange(0, T + 1, L, dtype=np.int64)
    return q, k, v, g, ts, torch.from_numpy(offs_h).to(dev), offs_h


w = torch.randn(16, device=dev) * 0.02
if "--once" in sys.argv:
    q, k, v, g, ts, offs, offs_h = case(16384, 2)
    for _ in range(2):
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, deterministic=False)
    torch.cuda.synchronize()
    sys.exit(0)
win_budget = os.environ.get("JH_WIN_BUDGET")
if os.environ.get("JH_WIN_CHUNK"):
    kernels.WINDOW_Q_CHUNK = int(os.environ["JH_WIN_CHUNK"])
only = os.environ.get("JH_ONLY")  # e.g. "windowed"
sizes = ((4096, 16), (16384, 4), (65536, 1), (262144, 1), (1 << 20, 1))
if len(sys.argv) > 1 and sys.argv[1].isdigit():
    sizes = sizes[:int(sys.argv[1])]
if len(sys.argv) > 2 and sys.argv[2].isdigit():
    sizes = sizes[int(sys.argv[2]):]
for L, B in sizes:
    q, k, v, g, ts, offs, offs_h = case(L, B)
    F = 5.0 * D * H * B * L * (L + 1)
    scratch = kernels.ds_scratch_bytes(H, offs_h)
    res = []
    reps = 3 if L <= 65536 else 1
    for name, det in (("fused", False), ("two-kernel", True), ("windowed", None)):
        if only and name not in only.split(","):
            continue
        if det and scratch > 24e9:
            res.append(f"two-kernel: scratch {scratch / 1e9:.1f} GB (skipped)")
            continue
        if det is None and win_budget:
            os.environ["JH_DS_SCRATCH_BUDGET"] = win_budget
        fn = lambda: kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, deterministic=det,  # noqa: E731
                                      seg_host=(offs_h, None, None))
        fn()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        os.environ.pop("JH_DS_SCRATCH_BUDGET", None)
        ms = e0.elapsed_time(e1) / reps
        peak = (torch.cuda.max_memory_allocated() - base) / 1e9
        res.append(f"{name}: {ms * 1e3:.0f} us {F / ms / 1e9:.0f} TF/s (extra peak {peak:.2f} GB)")
    print(f"L={L} B={B}: " + " | ".join(res), flush=True)
