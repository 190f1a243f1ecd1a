"""Do host->device and device->host copies overlap on this box (full-duplex PCIe)?"""
import time

import torch

dev = torch.device("cuda")
n = 64 << 20
a = torch.empty(n, dtype=torch.uint8).pin_memory()
b = torch.empty(n, dtype=torch.uint8).pin_memory()
da = torch.empty(n, dtype=torch.uint8, device=dev)
db = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    da.copy_(a, non_blocking=True)
    b.copy_(db, non_blocking=True)
torch.cuda.synchronize()


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / 10 * 1e3


def h2d():
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        b.copy_(db, non_blocking=True)


def both():
    h2d()
    d2h()


print(f"H2D {t(h2d):.3f} ms, D2H {t(d2h):.3f} ms, both on two streams {t(both):.3f} ms (64 MiB each)")
# slices of a pinned bf16 tensor, as the streaming API copies them
x = torch.randn(17526, 512).bfloat16().pin_memory()
r = 17526 // 4
print("slice is_pinned:", x[r:2 * r].is_pinned())


def slices():
    with torch.cuda.stream(s1):
        for i in range(4):
            x[i * r:(i + 1) * r].to(dev, non_blocking=True)


def whole():
    with torch.cuda.stream(s1):
        x.to(dev, non_blocking=True)


print(f"4 slice .to(): {t(slices):.3f} ms, whole .to(): {t(whole):.3f} ms ({x.numel() * 2 / 1e6:.1f} MB)")
xd = torch.empty_like(x, device=dev)


def slices_copy():
    with torch.cuda.stream(s1):
        for i in range(4):
            xd[i * r:(i + 1) * r].copy_(x[i * r:(i + 1) * r], non_blocking=True)


print(f"4 slice copy_ into preallocated: {t(slices_copy):.3f} ms")
