"""Device time (profiler) of norm_gate forward / backward on the C4 stack's
shapes (45105 rows, n = 512): gated with affine grads, plain with affine."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, '.')
from paper_2508_04711_b200 import _lib  # noqa: E402
from paper_2508_04711_b200 import kernels as k  # noqa: E402

if os.environ.get("JH_LIB"):  # A/B against another build (symbols it lacks are skipped)
    _lib.LIB_PATH = os.environ["JH_LIB"]
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in [s for s in _lib.SIGNATURES if not hasattr(L, s)]:
        del _lib.SIGNATURES[name]

rows, n = 45105, 512
x = torch.randn(rows, n, device='cuda').bfloat16()
uvqk = torch.randn(rows, 4 * n, device='cuda').bfloat16()
u = uvqk[:, :n]
dy = torch.randn_like(x)
gam = torch.randn(n, device='cuda')
bet = torch.randn(n, device='cuda')
y, mean, rstd = k.norm_gate_fwd(x, u, gam, bet)
fns = {"fwd gated": lambda: k.norm_gate_fwd(x, u, gam, bet), "fwd plain": lambda: k.norm_gate_fwd(x, None, gam, bet),
       "bwd gated": lambda: k.norm_gate_bwd(dy, x, u, gam, bet, mean, rstd),
       "bwd plain": lambda: k.norm_gate_bwd(dy, x, None, gam, bet, mean, rstd)}
for name, fn in fns.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
    per = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            per.setdefault(e.name[:32], []).append(e.time_range.elapsed_us())
    print(name + ": " + ", ".join(f"{n_} {sum(v) / len(v):.1f} us" for n_, v in per.items()), flush=True)
