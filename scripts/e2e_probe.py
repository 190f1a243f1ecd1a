"""Where the host-streaming e2e call spends its time (GPU box)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200.attention import hstu_attention_fwd_bwd_host  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=512, seed=7), 0)
pin = lambda a: torch.from_numpy(a).to(torch.bfloat16).pin_memory()  # noqa: E731
q, k, v = (pin(h[x]) for x in ("q", "k", "v"))
g = pin(np.random.default_rng(0).standard_normal(h["q"].shape).astype(np.float32))
ts = torch.from_numpy(h["ts"]).pin_memory()
w = np.random.default_rng(1).standard_normal(16) * 0.02
outs = [torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
dev = torch.device("cuda")
for G in (1, 2, 4, 8):
    for _ in range(3):
        hstu_attention_fwd_bwd_host(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G, out=outs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        hstu_attention_fwd_bwd_host(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G, out=outs)
    t1 = time.perf_counter()
    print(f"G={G}: {(t1 - t0) / 10 * 1e3:.3f} ms per call (wall)", flush=True)
# raw copy bandwidth for reference
x = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    x.copy_(q, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D {q.numel() * 2 / ((time.perf_counter() - t0) / 10) / 1e9:.1f} GB/s", flush=True)
t0 = time.perf_counter()
for _ in range(10):
    outs[0].copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H {q.numel() * 2 / ((time.perf_counter() - t0) / 10) / 1e9:.1f} GB/s", flush=True)
# host-side issue cost of one fwd + bwd call pair (device-resident inputs)
from paper_2508_04711_b200 import kernels  # noqa: E402
qd, kd, vd, gd = (x.to(dev) for x in (q, k, v, g))
tsd, od = ts.to(dev), torch.from_numpy(h["offsets"]).to(dev)
wd = torch.from_numpy(w.astype(np.float32)).to(dev)
for _ in range(3):
    kernels.attn_fwd(qd, kd, vd, tsd, tsd, od, 4, wd, 16)
    kernels.attn_bwd(qd, kd, vd, tsd, tsd, od, gd, 4, wd, 16, seg_host=(h["offsets"], None, None))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    kernels.attn_fwd(qd, kd, vd, tsd, tsd, od, 4, wd, 16)
t1 = time.perf_counter()
for _ in range(10):
    kernels.attn_bwd(qd, kd, vd, tsd, tsd, od, gd, 4, wd, 16, seg_host=(h["offsets"], None, None))
t2 = time.perf_counter()
torch.cuda.synchronize()
t3 = time.perf_counter()
print(f"host issue: fwd {(t1 - t0) / 10 * 1e6:.0f} us, bwd {(t2 - t1) / 10 * 1e6:.0f} us per call; "
      f"drain {(t3 - t2) * 1e3:.2f} ms", flush=True)
import cProfile  # noqa: E402
import pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    kernels.attn_bwd(qd, kd, vd, tsd, tsd, od, gd, 4, wd, 16, seg_host=(h["offsets"], None, None))
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
