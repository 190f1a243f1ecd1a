"""GPU checks of the HSTU layer: the row kernels (SiLU,
norm_gate) against torch fp32, and a 2-layer stack (bf16 kernels) against the
same stack in fp32 on torch ops with the oracle-bucketed dense attention
(tests/_layer_ref.py), forward and every gradient; the CP-sharded stack at
CP = 1 (one-rank NCCL group, resident-row path) against the plain stack.

Tolerances: row kernels 1e-2 relative to the row / column max (one bf16
rounding of the output); the stack 3e-2 row-normalised (bf16 activations at
every layer boundary, compounded over 2 layers), parameter gradients 3e-2 of
their max."""

import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from _cases import row_rel
from _layer_ref import TorchOps, copy_params

pytestmark = pytest.mark.gpu


def _k():
    from paper_2508_04711_b200 import kernels
    return kernels


def _rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return float((a - b).abs().max() / max(b.abs().max().item(), 1e-6))


def test_silu_fwd_bwd():
    g = torch.Generator(device="cuda").manual_seed(0)
    x = (3 * torch.randn(1000, 64, device="cuda", generator=g)).bfloat16()
    dy = torch.randn(1000, 64, device="cuda", generator=g).bfloat16()
    k = _k()
    y = k.silu(x)
    xr = x.float().requires_grad_(True)
    yr = F.silu(xr)
    yr.backward(dy.float())
    assert _rel(y, yr) <= 1e-2
    assert _rel(k.silu_bwd(x, dy), xr.grad) <= 1e-2


@pytest.mark.parametrize("rows,n", [(1, 8), (1000, 64), (333, 136), (45105, 2048), (700, 4096), (257, 8192)])
def test_silu_bwd_colsum_and_colsum(rows, n):
    # dx bitwise equal to the plain SiLU backward; the fused bias gradient and
    # jh_colsum against fp64 column sums of the same bf16 values (fp32
    # accumulation: 1e-5 of the column's absolute sum)
    g = torch.Generator(device="cuda").manual_seed(rows + n)
    x = (3 * torch.randn(rows, n, device="cuda", generator=g)).bfloat16()
    dy = torch.randn(rows, n, device="cuda", generator=g).bfloat16()
    k = _k()
    dx, db = k.silu_bwd_colsum(x, dy)
    assert torch.equal(dx, k.silu_bwd(x, dy))
    want = dx.double().sum(0)
    scale = dx.double().abs().sum(0) + 1e-30
    assert float(((db.double() - want).abs() / scale).max()) <= 1e-5
    # plain column sums of a strided view, added into an existing vector
    wide = torch.randn(rows, n + 24, device="cuda", generator=g).bfloat16()
    view = wide[:, 8:8 + n]
    out = torch.ones(n, device="cuda")
    k.colsum(view, out)
    want = view.double().sum(0) + 1
    scale = view.double().abs().sum(0) + 1
    assert float(((out.double() - want).abs() / scale).max()) <= 1e-5
    # deterministic
    assert torch.equal(k.silu_bwd_colsum(x, dy)[1], db)


@pytest.mark.parametrize("n,gate,affine", [(512, True, True), (512, False, True), (136, True, False),
                                           (2048, True, True)])
def test_norm_gate_fwd_bwd(n, gate, affine):
    rows = 777
    g = torch.Generator(device="cuda").manual_seed(n)
    x = (torch.randn(rows, n, device="cuda", generator=g) * 2 + 0.5).bfloat16()
    big = torch.randn(rows, 4 * n, device="cuda", generator=g).bfloat16()
    u = big[:, n:2 * n] if gate else None  # strided view, as in the layer
    gamma = (1 + 0.3 * torch.randn(n, device="cuda", generator=g)) if affine else None
    beta = 0.2 * torch.randn(n, device="cuda", generator=g) if affine else None
    dy = torch.randn(rows, n, device="cuda", generator=g).bfloat16()
    k = _k()
    y, mean, rstd = k.norm_gate_fwd(x, u, gamma, beta, 1e-6)
    dx, du, dg, db = k.norm_gate_bwd(dy, x, u, gamma, beta, mean, rstd)
    xr = x.float().requires_grad_(True)
    ur = u.float().requires_grad_(True) if gate else None
    gr = gamma.clone().requires_grad_(True) if affine else None
    br = beta.clone().requires_grad_(True) if affine else None
    yr = F.layer_norm(xr, (n,), gr, br, 1e-6)
    if gate:
        yr = yr * ur
    yr.backward(dy.float())
    assert _rel(y, yr) <= 1e-2
    assert row_rel(dx.float().cpu().numpy(), xr.grad.cpu().numpy())[1] <= 1e-2
    if gate:
        assert _rel(du, ur.grad) <= 1e-2
    if affine:
        assert _rel(dg, gr.grad) <= 1e-3
        assert _rel(db, br.grad) <= 1e-3


def _inputs(lens, E, seed):
    rng = np.random.default_rng(seed)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    x = torch.from_numpy(rng.standard_normal((T, E)).astype(np.float32)).bfloat16()
    ts = np.zeros(T, dtype=np.int64)
    for b, L in enumerate(lens):
        ts[offs[b]:offs[b] + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, 10**6, size=L))
    gy = torch.from_numpy(rng.standard_normal((T, E)).astype(np.float32)).bfloat16()
    return x, torch.from_numpy(ts), offs, gy


def _perturb(st):
    with torch.no_grad():
        for name, p in st.named_parameters():
            if "gamma" in name or "beta" in name or name.endswith("b_uvqk") or name.endswith("b_o"):
                p.add_(0.1 * torch.randn(p.shape, generator=torch.Generator().manual_seed(len(name))).to(p.device))


@pytest.mark.parametrize("lens,E,H,DH", [([300, 1, 130, 64], 256, 4, 64), ([513, 200], 512, 4, 128)])
def test_stack_matches_torch_fp32(lens, E, H, DH):
    from paper_2508_04711_b200.hstu_layer import HSTUStack
    x, ts, offs, gy = _inputs(lens, E, 3)
    st = HSTUStack(2, E, H, DH, 16, seed=1).cuda()
    _perturb(st)
    ref = HSTUStack(2, E, H, DH, 16, seed=1, ops=TorchOps).cuda()
    copy_params(ref, st)
    xg = x.cuda().requires_grad_(True)
    out = st(xg, ts.cuda(), torch.from_numpy(offs).cuda(), max(lens))
    out.backward(gy.cuda())
    TorchOps.offsets_host = offs
    try:
        xr = x.float().cuda().requires_grad_(True)
        outr = ref(xr, ts.cuda(), torch.from_numpy(offs).cuda(), max(lens))
        outr.backward(gy.float().cuda())
    finally:
        TorchOps.offsets_host = None
    torch.cuda.synchronize()
    e_out = row_rel(out.detach().float().cpu().numpy(), outr.detach().cpu().numpy())[1]
    e_dx = row_rel(xg.grad.float().cpu().numpy(), xr.grad.cpu().numpy())[1]
    print(f"stack out {e_out:.2e} dx {e_dx:.2e}")
    assert e_out <= 3e-2 and e_dx <= 3e-2
    for (name, p), (_, pr) in zip(st.named_parameters(), ref.named_parameters()):
        e = _rel(p.grad, pr.grad)
        print(f"  grad {name}: {e:.2e}")
        assert e <= 3e-2, name


def test_cp_stack_single_rank_matches_plain_stack():
    import torch.distributed as dist
    from paper_2508_04711_b200.cp_layer import CPAttention
    from paper_2508_04711_b200.hstu_layer import HSTUStack
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29700 + os.getpid() % 1000))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        lens = [300, 17, 129]
        E, H, DH = 256, 2, 128
        x, ts, offs, gy = _inputs(lens, E, 4)
        plain = HSTUStack(2, E, H, DH, 16, seed=2).cuda()
        cpst = HSTUStack(2, E, H, DH, 16, seed=2, cp=CPAttention(dist.group.WORLD, H, 16)).cuda()
        x1 = x.cuda().requires_grad_(True)
        o1 = plain(x1, ts.cuda(), torch.from_numpy(offs).cuda(), max(lens))
        o1.backward(gy.cuda())
        x2 = x.cuda().requires_grad_(True)
        o2 = cpst(x2, ts.cuda(), local_lengths=lens)
        o2.backward(gy.cuda())
        cpst.cp_grad_sync()
        torch.cuda.synchronize()
        assert row_rel(o2.detach().float().cpu().numpy(), o1.detach().float().cpu().numpy())[1] <= 2e-2
        assert row_rel(x2.grad.float().cpu().numpy(), x1.grad.float().cpu().numpy())[1] <= 2e-2
        for (name, p1), (_, p2) in zip(plain.named_parameters(), cpst.named_parameters()):
            assert _rel(p2.grad, p1.grad) <= 2e-2, name
    finally:
        dist.destroy_process_group()
