"""Rank 0 of the C4 stack at CP = 8 on this GPU (LoopbackComm: exchange
excluded): step time, GPU busy time and the top host / device ops.

NOT a timing of real CP: LoopbackComm fills the gathered K/V / timestamps
with replicas of this rank's rows, so the gathered timestamps are not the
sequence's (not monotone, small deltas) and the attention epilogues take the
slow exact-bucket paths instead of the saturated one.  Memory and the host /
plumbing costs are representative; attention kernel times are not."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2508_04711_b200.cp_layer import CPAttention, LoopbackComm  # noqa: E402
from paper_2508_04711_b200.hstu_layer import HSTUStack  # noqa: E402

dev = torch.device("cuda", 0)
lens, _ = bench._c4_batch()
cp_size = 8
per = lens.size // cp_size
ranks = [lens[r * per:(r + 1) * per] for r in range(cp_size)]
OVERLAP = os.environ.get("OVERLAP", "1") == "1"
cp = CPAttention(None, 4, 16, comm=LoopbackComm(cp_size, 0, peer_lengths=lambda r: ranks[r]), overlap=OVERLAP)
st = HSTUStack(8, 512, 4, 128, 16, seed=7, cp=cp).to(dev)
T0 = int(ranks[0].sum())
x = torch.randn(T0, 512, device=dev).bfloat16().requires_grad_(True)
gy = torch.randn(T0, 512, device=dev).bfloat16()
ts = torch.cumsum(torch.randint(1, 10**6, (T0,), device=dev), 0)


def step():
    x.grad = None
    st.zero_grad(set_to_none=True)
    st(x, ts, local_lengths=ranks[0]).backward(gy)


for _ in range(3):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    step()
e1.record()
torch.cuda.synchronize()
print(f"overlap={OVERLAP} step: events {e0.elapsed_time(e1) / 5:.2f} ms, wall {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms", flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ka = prof.key_averages()
print(ka.table(sort_by="cuda_time_total", row_limit=15), flush=True)
print(ka.table(sort_by="self_cpu_time_total", row_limit=15), flush=True)
