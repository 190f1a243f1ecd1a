"""Per-CTA busy time of each attention kernel on the C2 workload (load balance)."""
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
for _ in range(3):
    kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, bench.H, w, bench.NB, max_kv_len=bench.MAXLEN)
torch.cuda.synchronize()
for name in ("fwd", "bwd"):
    buf = torch.zeros(4096, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    kernels.set_trace(buf, -1)
    if name == "fwd":
        kernels.attn_fwd(q, k, v, ts, ts, offs, bench.H, w, bench.NB)
    else:
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, bench.H, w, bench.NB, max_kv_len=bench.MAXLEN)
    torch.cuda.synchronize()
    kernels.set_trace(None)
    raw = buf.cpu().numpy().astype(np.float64)
    bw0, bw1 = raw[3072], raw[3073]
    print(f"{name}: build_work {(bw1 - bw0) / 1e3:.1f} us")
    prev_end = bw1
    for kern in ([2] if name == "fwd" else [0, 1]):
        t = buf.cpu().numpy()[1024 * kern: 1024 * kern + 2 * 148].reshape(148, 2).astype(np.float64)
        t0 = t[:, 0].min()
        busy = (t[:, 1] - t[:, 0]) / 1e3
        end = (t[:, 1] - t0) / 1e3
        print(np.sort(busy).round(1))
        print(f"{name}[{kern}]: busy us min {busy.min():.1f} mean {busy.mean():.1f} max {busy.max():.1f}; "
              f"end us min {end.min():.1f} max {end.max():.1f}; start spread {(t[:, 0].max() - t0) / 1e3:.1f}; "
              f"gap from previous kernel's end {(t0 - prev_end) / 1e3:.1f}")
        prev_end = t[:, 1].max()
