"""Steady-state cost per tile / half: long segments (diagonal blocks are a small
fraction), large time gaps (off-diagonal chunks saturated).  Prints the fwd and
bwd kernel times and the implied SM cycles per fwd tile and per dK/dV half."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402

L, B, H, D = int(os.environ.get("L", 8192)), int(os.environ.get("B", 4)), 4, 128
torch.manual_seed(0)
dev = "cuda"
T = L * B
q, k, v, g = (torch.randn(T, H * D, device=dev).bfloat16() for _ in range(4))
gaps = torch.randint(100_000, 1_000_000, (T,), device=dev)
ts = torch.cumsum(gaps, 0)
offs = torch.arange(0, T + 1, L, device=dev, dtype=torch.int64)
w = torch.randn(16, device=dev) * 0.02
for _ in range(3):
    kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=(offs.cpu().numpy(), None, None))
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
for _ in range(5):
    kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16)
ev[1].record()
for _ in range(5):
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=(offs.cpu().numpy(), None, None))
ev[2].record()
torch.cuda.synchronize()
tf, tb = ev[0].elapsed_time(ev[1]) / 5, ev[1].elapsed_time(ev[2]) / 5
nq = (L + 127) // 128
tiles = B * H * nq * (nq + 1) // 2
halves = B * H * sum(2 * nq - 2 * j for j in range(nq))
clk = 1.965e6  # cycles per ms
F = 2.0 * D * H * B * L * (L + 1)
print(f"[{'fwd2' if os.environ.get('JH_FWD2') == '1' else 'fwd1'}] L={L} B={B}: fwd {tf * 1e3:.1f} us "
      f"({F / tf / 1e9:.0f} TF/s)  ({tf * clk * 148 / tiles:.0f} cycles/tile/SM)   "
      f"bwd {tb * 1e3:.1f} us  ({tb * clk * 148 / halves:.0f} cycles/half/SM incl. dQ)")
