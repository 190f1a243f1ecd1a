"""Wall time of the host-streaming e2e call per run count G (r2: 2.45-2.5 ms for
G = 2..6 whatever the split; first / last runs at 0.25-1x the middle ones made
no difference -- the PCIe rates, ~42 GB/s per direction while both run, bind)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import attention  # noqa: E402
from paper_2508_04711_b200.harness import ExperimentConfig, gen_synthetic_host  # noqa: E402

h = gen_synthetic_host(ExperimentConfig(cp_size=1, batch_size=32, min_len=1, max_len=1024, max_length=1024,
                                        embed_dim=512, seed=7), 0)
pin = lambda a: torch.from_numpy(a).to(torch.bfloat16).pin_memory()  # noqa: E731
q, k, v = (pin(h[x]) for x in ("q", "k", "v"))
g = pin(np.random.default_rng(0).standard_normal(h["q"].shape).astype(np.float32))
ts = torch.from_numpy(h["ts"]).pin_memory()
w = np.random.default_rng(1).standard_normal(16) * 0.02
outs = [torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
for rep in range(2):
    for e in (1.0,):
        row = []
        for G in (2, 3, 4, 6, 8):
            for _ in range(3):
                attention.hstu_attention_fwd_bwd_host(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G, out=outs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(20):
                attention.hstu_attention_fwd_bwd_host(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G, out=outs)
            row.append(f"G={G} {(time.perf_counter() - t0) / 20 * 1e3:.3f}")
        print(f"edge {e}: " + "  ".join(row), flush=True)

# back-to-back async calls (two output buffer sets), per G
outs2 = [torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=True) for _ in range(4)]
row = []
for G in (1, 2, 3, 4):
    sets = (outs, outs2)
    for i in range(4):
        attention.hstu_attention_fwd_bwd_host_async(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G,
                                                    out=sets[i % 2]).wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prev = None
    for i in range(20):
        cur = attention.hstu_attention_fwd_bwd_host_async(q, k, v, ts, h["offsets"], g, w, 4, 16, groups=G,
                                                          out=sets[i % 2])
        if prev is not None:
            prev.wait()
        prev = cur
    prev.wait()
    row.append(f"G={G} {(time.perf_counter() - t0) / 20 * 1e3:.3f}")
print("pipelined: " + "  ".join(row), flush=True)
