"""Device time of the attention calls on a trivial input (launch/setup overhead)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402

dev = "cuda"
H, D = 4, 128
for T in (1, 1024):
    q = torch.randn(T, H * D, device=dev).bfloat16()
    k, v, g = q.clone(), q.clone(), q.clone()
    ts = torch.arange(T, device=dev, dtype=torch.int64) * 1000
    offs = torch.tensor([0, T], device=dev, dtype=torch.int64)
    w = torch.randn(16, device=dev) * 0.02
    for _ in range(5):
        kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16)
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, max_kv_len=T)
    torch.cuda.synchronize()
    N = 50
    pf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    pb = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    big = torch.empty(64 << 20, device=dev)
    big.fill_(1.0)  # keep the GPU busy while the host enqueues
    for i in range(N):
        kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, prof=pf[i])
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, prof=pb[i], max_kv_len=T)
    torch.cuda.synchronize()
    f = np.median([a.elapsed_time(b) for a, b in pf]) * 1e3
    b = np.median([a.elapsed_time(b) for a, b in pb]) * 1e3
    print(f"T={T}: fwd kernel {f:.1f} us, bwd kernels {b:.1f} us (event pairs around the kernels)")
