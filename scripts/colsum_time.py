"""Device time (profiler) of the SiLU-backward + bias column sum vs the plain
SiLU backward and torch's column reduction on the C4 stack's uvqk shape."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2508_04711_b200 import kernels as k  # noqa: E402

x = torch.randn(45105, 2048, device='cuda').bfloat16()
dy = torch.randn_like(x)
y = x[:, :512].contiguous()
fns = {"silu_bwd": lambda: k.silu_bwd(x, dy), "silu_bwd_colsum": lambda: k.silu_bwd_colsum(x, dy),
       "torch sum 2048": lambda: x.sum(0), "colsum 512": lambda: k.colsum(y), "torch sum 512": lambda: y.sum(0)}
for name, fn in fns.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    per = {}
    for e in evs:
        per.setdefault(e.name[:40], []).append(e.time_range.elapsed_us())
    print(name + ": " + ", ".join(f"{n} {sum(v) / len(v):.1f} us" for n, v in per.items()), flush=True)
