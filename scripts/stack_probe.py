"""8-layer HSTU stack on the C4 batch: eager step vs the same step captured
in a CUDA graph (host launch overhead), and the attention share (GPU box)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_04711_b200.hstu_layer import HSTUStack  # noqa: E402

dev = torch.device("cuda")
lens, ts_h = bench._c4_batch()
offs_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
T = int(offs_h[-1])
st = HSTUStack(8, 512, 4, 128, 16, seed=7).to(dev)
x = torch.randn(T, 512, device=dev).bfloat16().requires_grad_(True)
gy = torch.randn(T, 512, device=dev).bfloat16()
ts, offs = torch.from_numpy(ts_h).to(dev), torch.from_numpy(offs_h).to(dev)
maxlen = int(lens.max())


def step():
    st(x, ts, offs, maxlen).backward(gy)


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print(f"eager step {timed(step):.2f} ms", flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14), flush=True)
