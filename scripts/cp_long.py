"""One rank's share of a long single sequence through CPAttention (forward +
backward, LoopbackComm: communication excluded) -- the windowed two-kernel
backward vs the fused kernel for the long remote segments.
usage: python scripts/cp_long.py [L] [cp]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402
from paper_2508_04711_b200.cp_layer import CPAttention, LoopbackComm  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
cp_size = int(sys.argv[2]) if len(sys.argv) > 2 else 8
H, D = 4, 128
dev = torch.device("cuda", 0)
cp = CPAttention(None, H, 16, comm=LoopbackComm(cp_size, 0, peer_lengths=lambda r: []))
p, pd = cp.plan_for([L], dev)
n = p.n_res
gen = torch.Generator(device=dev).manual_seed(1)
q, k, v, g = (torch.randn(n, H * D, device=dev, generator=gen).bfloat16() for _ in range(4))
ts = torch.cumsum(torch.randint(1, 10**6, (n,), device=dev, generator=gen), 0)
w = torch.randn(16, device=dev) * 0.02
F = 7.0 * D * H * L * (L + 1) / cp_size  # one rank's share of the causal flops (fwd 2 + bwd 5)
for enabled in (False, True, False, True):
    kernels.WINDOWED_BWD["enabled"] = enabled
    o, ctx = cp.attend(q, k, v, ts, p, pd, w)
    cp.attend_backward(ctx, g, w)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    o, ctx = cp.attend(q, k, v, ts, p, pd, w)
    cp.attend_backward(ctx, g, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"L={L} cp={cp_size} rank rows={n} windowed={enabled}: fwd+bwd {ms:.1f} ms, {F / ms / 1e9:.0f} TF/s "
          f"(wall {1e3 * (time.perf_counter() - t0):.0f} ms)", flush=True)
