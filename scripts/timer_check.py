"""globaltimer vs clock64 vs CUDA events for the forward kernel (bench conditions)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_04711_b200 import kernels  # noqa: E402

h = bench._host_batch(0)
dev = "cuda"
q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
w = torch.from_numpy(bench._ts_weights().astype(np.float32)).to(dev)
for _ in range(3):
    kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
torch.cuda.synchronize()
big = torch.empty(256 << 20, device=dev)
buf = torch.zeros(4096, dtype=torch.int64, device=dev)
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
big.fill_(1.0)
kernels.set_trace(buf, -1)
kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB, prof=ev)
kernels.set_trace(None)
torch.cuda.synchronize()
r = buf.cpu().numpy().astype(np.float64)
gt = r[2048:2048 + 296].reshape(148, 2)
ck = r[2048 + 512:2048 + 512 + 296].reshape(148, 2)
print("event us", ev[0].elapsed_time(ev[1]) * 1e3)
print("globaltimer span us (first start .. last end)", (gt[:, 1].max() - gt[:, 0].min()) / 1e3)
print("CTA0 globaltimer us", (gt[0, 1] - gt[0, 0]) / 1e3, " clock64 cycles", ck[0, 1] - ck[0, 0],
      " -> MHz", (ck[0, 1] - ck[0, 0]) / ((gt[0, 1] - gt[0, 0]) / 1e3))
