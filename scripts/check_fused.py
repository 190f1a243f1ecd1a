"""Quick GPU check of the fused backward against the oracle (GPU box)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
from _cases import make_case, row_rel, synthetic  # noqa: E402
from paper_2508_04711_b200 import kernels  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "small"
if which == "small":
    lens, H, d = [1, 130, 257, 64], 1, 128
elif which == "ragged":
    lens, H, d = [5, 0, 17, 1, 32, 129, 255, 256, 257], 2, 64
elif which == "mid":
    lens, H, d = [300, 77, 1000], 4, 128
else:
    lens, H, d = None, 4, 128
if lens is None:
    b = synthetic(7, 0, 32, 1024, 4, 128)
    case = dict(q=b["q"], k=b["k"], v=b["v"], g=b["q"][::-1].copy(), ts=b["ts"], offsets=b["offsets"],
                w=oracle.normal_init_ts_weights(16, 7 + 0x5EED), nb=16)
else:
    case = make_case(lens, H * d, seed=3)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
c = {x: t(case[x]).bfloat16() for x in ("q", "k", "v", "g")}
w = t(np.asarray(case["w"], np.float32))
for det in (False, True, False):
    t0 = time.time()
    dq, dk, dv, dw, _ = kernels.attn_bwd(c["q"], c["k"], c["v"], t(case["ts"]), t(case["ts"]), t(case["offsets"]),
                                         c["g"], H, w, 16, deterministic=det)
    torch.cuda.synchronize()
    print(f"{which} det={det} time {time.time() - t0:.3f}s", flush=True)
    wq, wk, wv, ww, _ = oracle.hstu_backward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["g"],
                                             case["w"], 16, H)
    for name, a, b in (("dq", dq, wq), ("dk", dk, wk), ("dv", dv, wv)):
        print(f"  {name}: max_abs/row_rel = {row_rel(a.float().cpu().numpy(), b)}", flush=True)
    dwn = dw.cpu().numpy()
    print(f"  dw rel {np.abs(dwn - ww).max() / np.abs(ww).max():.3e}", flush=True)
