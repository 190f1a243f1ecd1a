"""Device timeline (torch profiler / CUPTI) of one host-streaming e2e call:
start / end of every memcpy and kernel, relative to the first activity."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200.attention import hstu_attention_fwd_bwd_host  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=512, seed=7), 0)
pin = lambda a: torch.from_numpy(a).to(torch.bfloat16).pin_memory()  # noqa: E731
q, k, v = (pin(h[x]) for x in ("q", "k", "v"))
g = pin(np.random.default_rng(0).standard_normal(h["q"].shape).astype(np.float32))
ts = torch.from_numpy(h["ts"]).pin_memory()
w = np.random.default_rng(1).standard_normal(16) * 0.02
outs = [torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
for _ in range(5):
    hstu_attention_fwd_bwd_host(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G, out=outs)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    hstu_attention_fwd_bwd_host(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G, out=outs)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0):8.1f} {(e.time_range.end - t0):8.1f} {e.time_range.elapsed_us():7.1f}  "
          f"{e.name[:70]}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
c0 = min(e.time_range.start for e in cpu)
print("host span", max(e.time_range.end for e in cpu) - c0, "us; first device activity at", t0 - c0)
