"""Small shapes through every kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck): fused forward, both backward paths, the
CP segment form, the bandwidth helpers and the HSTU-layer row kernels."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402

dev = "cuda"
H, D = 2, 128
lens = [1, 130, 257, 64, 0, 300]
offs_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
T = int(offs_h[-1])
torch.manual_seed(0)
q, k, v, g = (torch.randn(T, H * D, device=dev).bfloat16() for _ in range(4))
ts = torch.cumsum(torch.randint(1, 10**5, (T,), device=dev), 0)
offs = torch.from_numpy(offs_h).to(dev)
w = torch.randn(16, device=dev) * 0.02
band = kernels.new_band_table(T, len(lens), q.device)
kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band)
for det in (True, False):
    kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, band_table=band, deterministic=det,
                     seg_host=(offs_h, None, None))
# segment (CP remote) form, fp32 partials
qo = torch.tensor([0, 100], device=dev)
acc = torch.zeros(100, H * D, device=dev)
kernels.attn_fwd(q[200:300].contiguous(), k, v, ts[200:300].contiguous(), ts, qo, H, w, 16,
                 q_pos0=torch.tensor([200], device=dev), kv_start=torch.tensor([0], device=dev),
                 kv_len=torch.tensor([200], device=dev), kv_len_total=200, out_accum=acc)
# helpers and layer kernels
perm = torch.randperm(T, device=dev)
kernels.gather_rows(q, perm)
kernels.bucketize(torch.randint(-5, 10**7, (4096,), device=dev), 16)
x = torch.randn(T, 512, device=dev).bfloat16()
y, m, r = kernels.norm_gate_fwd(x, x, torch.ones(512, device=dev), torch.zeros(512, device=dev))
kernels.norm_gate_bwd(y, x, x, torch.ones(512, device=dev), torch.zeros(512, device=dev), m, r)
kernels.silu_bwd(x, kernels.silu(x))
torch.cuda.synchronize()
print("sanitize smoke done")
