"""C2 step with the forward and the backward on two streams (the HSTU backward
recomputes from q, k, v and never reads the forward's output) vs the same two
calls back to back on one stream: CUDA-graph replays, L2 flushed between."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

H = 4
dev = torch.device("cuda", 0)
h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=512, seed=7), 0)
q, k, v = (torch.from_numpy(h[x]).to(dev).bfloat16() for x in ("q", "k", "v"))
ts = torch.from_numpy(h["ts"]).to(dev)
offs = torch.from_numpy(h["offsets"]).to(dev)
g = torch.randn_like(q)
w = torch.randn(16, device=dev) * 0.02
seg = (h["offsets"], None, None)
band_f = kernels.new_band_table(q.shape[0], offs.numel() - 1, dev)
band_b = kernels.new_band_table(q.shape[0], offs.numel() - 1, dev)
kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band_b)  # band_b computed once, reused ready
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
PRI = os.environ.get("PRI", "0,0").split(",")  # stream priorities (fwd, bwd): lower = higher priority
sf, sb = torch.cuda.Stream(dev, priority=int(PRI[0])), torch.cuda.Stream(dev, priority=int(PRI[1]))


def serial():
    kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band_f)
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=seg, band_table=band_f)


def two_streams(first_bwd=False):
    main = torch.cuda.current_stream(dev)
    sf.wait_stream(main)
    sb.wait_stream(main)
    order = [(sb, "b"), (sf, "f")] if first_bwd else [(sf, "f"), (sb, "b")]
    for s, which in order:
        with torch.cuda.stream(s):
            if which == "f":
                kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band_f)
            else:
                kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, seg_host=seg, band_table=band_b)
    main.wait_stream(sf)
    main.wait_stream(sb)


def graph_time(fn, n=30):
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream(dev).wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    tot = 0.0
    for i in range(n):
        flush.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3


for rep in range(2):
    print(f"[prio fwd,bwd = {PRI}] serial {graph_time(serial):.1f} us | fwd || bwd (fwd first) {graph_time(two_streams):.1f} us | "
          f"(bwd first) {graph_time(lambda: two_streams(True)):.1f} us", flush=True)

# the batch split into two halves of whole sequences, each half's fwd || bwd on its own stream pair
import numpy as np  # noqa: E402
offs_h = h["offsets"]
B = offs_h.size - 1
cut = int(np.searchsorted(offs_h, offs_h[-1] / 2))
halves = []
for b0, b1 in ((0, cut), (cut, B)):
    r0, r1 = int(offs_h[b0]), int(offs_h[b1])
    sub = offs_h[b0:b1 + 1] - r0
    halves.append(dict(q=q[r0:r1], k=k[r0:r1], v=v[r0:r1], g=g[r0:r1], ts=ts[r0:r1].clone(),
                       o=torch.from_numpy(sub).to(dev), seg=(sub, None, None),
                       band=kernels.new_band_table(r1 - r0, b1 - b0, dev)))
side = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]


def split_step():
    main = torch.cuda.current_stream(dev)
    for s_, hh in zip(side, halves):
        s_.wait_stream(main)
        with torch.cuda.stream(s_):
            kernels.attn_fwd_bwd(hh["q"], hh["k"], hh["v"], hh["ts"], hh["o"], hh["g"], H, w, 16, seg_host=hh["seg"],
                                 band_table=hh["band"])
    for s_ in side:
        main.wait_stream(s_)


def full_step():
    kernels.attn_fwd_bwd(q, k, v, ts, offs, g, H, w, 16, seg_host=seg, band_table=band_f)


for rep in range(2):
    print(f"attn_fwd_bwd full batch {graph_time(full_step):.1f} us | two halves on two stream pairs "
          f"{graph_time(split_step):.1f} us", flush=True)
