"""Record the per-role device timeline of the fused kernels on the C2
workload (one CTA) and print it as (role, event, arg, cycles since start)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
H, D = 4, 128
dev = "cuda"
if os.environ.get("L"):  # steady-state workload: B segments of length L, large time gaps
    L, B = int(os.environ["L"]), int(os.environ.get("B", 4))
    torch.manual_seed(0)
    q, k, v = (torch.randn(L * B, H * D, device=dev).bfloat16() for _ in range(3))
    ts = torch.cumsum(torch.randint(100_000, 1_000_000, (L * B,), device=dev), 0)
    offs = torch.arange(0, L * B + 1, L, device=dev, dtype=torch.int64)
else:
    h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                            embed_dim=H * D, seed=7), 0)
    q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
    ts = torch.from_numpy(h["ts"]).to(dev)
    offs = torch.from_numpy(h["offsets"]).to(dev)
g = torch.randn_like(q)
w = torch.randn(16, device=dev) * 0.02
for _ in range(3):
    kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, max_kv_len=int(os.environ.get('L', 1024)))
torch.cuda.synchronize()
out = {}
for name in ("fwd", "bwd"):
    buf = torch.zeros(5 * 4096 * 2, dtype=torch.int64, device=dev)
    kernels.set_trace(buf, cta)
    if name == "fwd":
        kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16)
    else:
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, max_kv_len=int(os.environ.get('L', 1024)))
    torch.cuda.synchronize()
    kernels.set_trace(None)
    t = buf.view(5, 4096, 2).cpu().numpy()
    ev = []
    for role in range(5):
        for i in range(4096):
            tag, clk = int(t[role, i, 0]), int(t[role, i, 1])
            if clk == 0:
                break
            ev.append((clk, role, tag >> 32, tag & 0xFFFFFFFF))
    ev.sort()
    t0 = ev[0][0] if ev else 0
    out[name] = [(c - t0, r, code, arg) for c, r, code, arg in ev]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"trace_cta{cta}.json"), "w") as f:
    json.dump(out, f)
for name, evs in out.items():
    print(name, "events", len(evs), "span cycles", evs[-1][0] if evs else 0)
