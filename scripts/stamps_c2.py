"""Per-CTA start / end stamps (globaltimer + clock64) of the attention kernels
on C2, plus the one-CTA role timeline of the forward: load balance and
per-item overhead.  python scripts/stamps_c2.py -> gpurun_out/stamps_c2.json"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

H, D = 4, 128
dev = "cuda"
h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=H * D, seed=7), 0)
q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
g = torch.randn_like(q)
w = torch.randn(16, device=dev) * 0.02
seg = (h["offsets"], None, None)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
band = kernels.new_band_table(q.shape[0], offs.numel() - 1, q.device)
for _ in range(3):
    kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=seg, band_table=band)
torch.cuda.synchronize()
res = {}
for name in ("fwd", "bwd"):
    buf = torch.zeros(4 * 1024, dtype=torch.int64, device=dev)
    flush.zero_()
    kernels.set_trace(buf, -1)
    if name == "fwd":
        kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band)
    else:
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=seg, band_table=band)
    torch.cuda.synchronize()
    kernels.set_trace(None)
    t = buf.cpu().numpy()
    for kk in range(3):
        base = 1024 * kk
        st, en = t[base:base + 296:2], t[base + 1:base + 296:2]
        if (st == 0).all():
            continue
        m = st > 0
        t0 = st[m].min()
        res[f"{name}_k{kk}"] = {"start_ns": (st[m] - t0).tolist(), "end_ns": (en[m] - t0).tolist()}
        print(f"{name} kernel{kk}: CTAs {m.sum()} start spread {(st[m]-t0).max()/1e3:.1f} us, end min/med/max "
              f"{(en[m]-t0).min()/1e3:.1f}/{np.median(en[m]-t0)/1e3:.1f}/{(en[m]-t0).max()/1e3:.1f} us", flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "stamps_c2.json"), "w") as f:
    json.dump(res, f)
