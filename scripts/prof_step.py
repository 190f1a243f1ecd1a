"""GPU timeline of the C2 bench step (torch.profiler / CUPTI): every kernel and
memcpy/memset on the device with its duration, and the idle gaps between them."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_04711_b200 import kernels  # noqa: E402

h = bench._host_batch(0)
T = int(h["offsets"][-1])
dev = "cuda"
q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
g = torch.randn_like(q)
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
w = torch.from_numpy(bench._ts_weights().astype(np.float32)).to(dev)


def step():
    kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
    return kernels.attn_bwd(q, k, v, ts, ts, offs, g, bench.H, w, bench.NB)


for _ in range(5):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
for e in evs:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    print(f"{s - t0:9.1f} us  gap {s - prev_end:7.1f}  dur {d:8.1f}  {e.name[:90]}")
    prev_end = e.time_range.end
cpu = [e for e in prof.events() if e.device_type.name == "CPU" and e.name.startswith("aten::")]
print("cpu ops per 3 steps:", len(cpu))
