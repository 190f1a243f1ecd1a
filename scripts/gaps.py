"""Kernel boundary gaps of one fwd+bwd step (globaltimer stamps, trace_cta = -1)."""
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
g = torch.randn_like(q)
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
w = torch.from_numpy(bench._ts_weights().astype(np.float32)).to(dev)


def step():
    kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, bench.H, w, bench.NB, max_kv_len=bench.MAXLEN)


for _ in range(3):
    step()
torch.cuda.synchronize()
buf = torch.zeros(4096, dtype=torch.int64, device=dev)
kernels.set_trace(buf, -1)
step()
torch.cuda.synchronize()
kernels.set_trace(None)
r = buf.cpu().numpy().astype(np.float64)
fwd = r[2048:2048 + 296].reshape(148, 2)
dkv = r[0:296].reshape(148, 2)
dq = r[1024:1024 + 296].reshape(148, 2)
t0 = fwd[:, 0].min()
for name, a in (("fwd", fwd), ("dkv", dkv), ("dq", dq)):
    print(f"{name}: first start {(a[:, 0].min() - t0) / 1e3:8.1f}  last start {(a[:, 0].max() - t0) / 1e3:8.1f}  "
          f"first end {(a[:, 1].min() - t0) / 1e3:8.1f}  last end {(a[:, 1].max() - t0) / 1e3:8.1f}")
print(f"bwd build_work: {(r[3072] - t0) / 1e3:.1f} .. {(r[3073] - t0) / 1e3:.1f}")

cyc = r[512:512 + 296].reshape(148, 2)
halves = cyc[:, 0]
busy = (dkv[:, 1] - dkv[:, 0]) / 1e3
order = np.argsort(busy)
print("dkv CTAs (busy us, halves): fastest", [(round(busy[i], 1), int(halves[i])) for i in order[:5]],
      "slowest", [(round(busy[i], 1), int(halves[i])) for i in order[-5:]])
print("halves per CTA min/mean/max", halves.min(), halves.mean(), halves.max())
