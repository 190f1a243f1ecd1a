"""Kernel timings on the C2 workload (GPU box): python scripts/time_c2.py
Times the forward and the backward variants with CUDA events (L2 flushed
between reps).  JH_DBG bits (fused backward timing experiments): 8 = no dQ
reductions, 16 = no epilogue math."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _cases import synthetic  # noqa: E402
import oracle  # noqa: E402
from paper_2508_04711_b200 import kernels  # noqa: E402

H, D = 4, 128
b = synthetic(7, 0, 32, 1024, H, D)
dev = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
q, k, v = (t(b[x]).bfloat16() for x in ("q", "k", "v"))
g = t(b["q"][::-1].copy()).bfloat16()
ts, offs = t(b["ts"]), t(b["offsets"])
w = t(oracle.normal_init_ts_weights(16, 7 + 0x5EED).astype(np.float32))
L = np.diff(b["offsets"])
F_fwd = 2 * D * H * float((L * (L + 1)).sum())
F_bwd = 2.5 * F_fwd
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1))
    return float(np.median(tot))


band = kernels.new_band_table(q.shape[0], offs.numel() - 1, q.device)
ms = timeit(lambda: kernels.attn_fwd(q, k, v, ts, ts, offs, H, w, 16, band_table=band))
print(f"fwd ({'fwd2' if os.environ.get('JH_FWD2') == '1' else 'fwd1'}): {ms * 1e3:.1f} us  "
      f"{F_fwd / ms / 1e9:.1f} TF/s  frac {F_fwd / ms / 1e9 / 1650.2:.3f}", flush=True)
if os.environ.get("JH_FWD2") != "1":
    for det, dbg in ((True, 0),) if os.environ.get("JH_ALL") != "1" else ((True, 0), (False, 0), (False, 8), (False, 16), (False, 24)):
        os.environ["JH_DBG"] = str(dbg)
        ms = timeit(lambda: kernels.attn_bwd(q, k, v, ts, ts, offs, g, H, w, 16, band_table=band,
                                             deterministic=det, max_kv_len=int(L.max())))
        print(f"bwd det={det} dbg={dbg}: {ms * 1e3:.1f} us  {F_bwd / ms / 1e9:.1f} TF/s  frac "
              f"{F_bwd / ms / 1e9 / 1650.2:.3f}", flush=True)
    os.environ["JH_DBG"] = "0"
