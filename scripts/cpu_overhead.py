"""Host (enqueue) time of the fwd / bwd calls, and GPU time of a CUDA-graph replay."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_04711_b200 import kernels  # noqa: E402

h = bench._host_batch(0)
dev = "cuda"
q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
g = torch.randn_like(q)
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
w = torch.from_numpy(bench._ts_weights().astype(np.float32)).to(dev)
for _ in range(5):
    kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, bench.H, w, bench.NB, max_kv_len=bench.MAXLEN)
torch.cuda.synchronize()
N = 50
tf = tb = 0.0
for _ in range(N):
    t0 = time.perf_counter()
    kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
    t1 = time.perf_counter()
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, bench.H, w, bench.NB, max_kv_len=bench.MAXLEN)
    t2 = time.perf_counter()
    tf += t1 - t0
    tb += t2 - t1
    torch.cuda.synchronize()
print(f"host enqueue: fwd {tf / N * 1e6:.1f} us  bwd {tb / N * 1e6:.1f} us")
