"""Gaps between the kernels of one C2 fwd+bwd step (globaltimer CTA stamps,
both calls enqueued back to back as in the bench): fwd end -> dK/dV start."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

H = 4
dev = "cuda"
h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=512, seed=7), 0)
q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
g = torch.randn_like(q)
w = torch.randn(16, device=dev) * 0.02
seg = (h["offsets"], None, None)
band = kernels.new_band_table(q.shape[0], offs.numel() - 1, q.device)


def step():
    if os.environ.get("SERIAL"):
        kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band)
        kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=seg, band_table=band)
    else:  # the bench's step: band table, then forward || backward on two streams
        kernels.attn_fwd_bwd(q, k, v, ts, offs, g, H, w, 16, seg_host=seg, band_table=band)


for _ in range(3):
    step()
torch.cuda.synchronize()
buf = torch.zeros(4 * 1024, dtype=torch.int64, device=dev)
kernels.set_trace(buf, -1)  # baked into the captured launches
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
kernels.set_trace(None)
for rep in range(3):
    buf.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    t = buf.cpu().numpy()
    st = {kk: t[1024 * kk:1024 * kk + 296:2] for kk in range(3)}
    en = {kk: t[1024 * kk + 1:1024 * kk + 296:2] for kk in range(3)}
    t0 = min(x[x > 0].min() for x in st.values())
    f = lambda a: (a[a > 0] - t0) / 1e3  # noqa: E731
    print(f"rep {rep}: step {e0.elapsed_time(e1) * 1e3:.1f} us | fwd {f(st[2]).min():.1f}-{f(en[2]).max():.1f} | "
          f"dkv {f(st[0]).min():.1f}-{f(en[0]).max():.1f} | dq {f(st[1]).min():.1f}-{f(en[1]).max():.1f} us",
          flush=True)
