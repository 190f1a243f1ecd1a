"""Per-step wall times of back-to-back async host-streaming calls (C2 batch),
with device / pinned-host allocator statistics: diagnoses stalls in the
pipelined e2e leg."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import attention  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=512, seed=7), 0)
pin = lambda a: torch.from_numpy(a).to(torch.bfloat16).pin_memory()  # noqa: E731
q, k, v = (pin(h[x]) for x in ("q", "k", "v"))
g = pin(np.random.default_rng(0).standard_normal(h["q"].shape).astype(np.float32))
ts = torch.from_numpy(h["ts"]).pin_memory()
w = np.random.default_rng(1).standard_normal(16) * 0.02
sets = [[torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)] for _ in range(2)]
for i in range(3):
    attention.hstu_attention_fwd_bwd_host_async(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=2,
                                                out=sets[i % 2]).wait()
torch.cuda.synchronize()
prev = None
t_last = time.perf_counter()
times, submit = [], []
for i in range(K):
    t_s = time.perf_counter()
    cur = attention.hstu_attention_fwd_bwd_host_async(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=2,
                                                      out=sets[i % 2])
    submit.append((time.perf_counter() - t_s) * 1e3)
    if prev is not None:
        prev.wait()
    prev = cur
    t = time.perf_counter()
    times.append((t - t_last) * 1e3)
    t_last = t
prev.wait()
print("per-step ms:", " ".join(f"{x:.2f}" for x in times))
print(f"host submit ms: mean {np.mean(submit):.3f} max {np.max(submit):.3f}")
print("reserved GB", torch.cuda.memory_reserved() / 1e9, "num_alloc_retries",
      torch.cuda.memory_stats().get("num_alloc_retries"))
try:
    print("host stats", {k_: v_ for k_, v_ in torch.cuda.host_memory_stats().items() if "alloc" in k_ and "num" in k_})
except Exception as e:  # noqa: BLE001
    print("no host stats", e)
