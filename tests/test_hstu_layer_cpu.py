"""HSTU layer / stack host logic on CPU: the CP-sharded stack (activations
redistributed once, resident across layers, restored once; K/V exchanged per
layer) equals the single-device stack on the concatenated batch, forward and
all parameter gradients, at world sizes 2 and 3 over gloo (fp64, the row ops
and attention on the torch / numpy doubles)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from _layer_ref import TorchOps, copy_params
from test_cp_gloo import NumpyBackend


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


E, H, DH, NL = 16, 2, 8, 2


def _batch(rank, lens):
    rng = np.random.default_rng([21, rank])
    T = int(sum(lens))
    x = rng.standard_normal((T, E))
    ts = np.zeros(T, dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    for b, L in enumerate(lens):
        ts[offs[b]:offs[b] + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, 10**6, size=L))
    g = rng.standard_normal((T, E))
    return x, ts, g


def _stack(cp=None):
    from paper_2508_04711_b200.hstu_layer import HSTUStack
    st = HSTUStack(NL, E, H, DH, 16, seed=5, cp=cp, ops=TorchOps).double()
    with torch.no_grad():  # non-trivial affine parameters
        for name, p in st.named_parameters():
            if "gamma" in name or "beta" in name or name.endswith("b_uvqk") or name.endswith("b_o"):
                p.add_(0.1 * torch.randn(p.shape, generator=torch.Generator().manual_seed(len(name)),
                                         dtype=p.dtype))
    return st


def _worker(rank, world, port, lens, result_dir, retain):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04711_b200.cp_layer import CPAttention
    cp = CPAttention(dist.group.WORLD, H, 16, backend=NumpyBackend(), retain_kv=retain)
    st = _stack(cp)
    x, ts, g = _batch(rank, lens[rank])
    xt = torch.from_numpy(x).requires_grad_(True)
    out = st(xt, torch.from_numpy(ts), local_lengths=lens[rank])
    out.backward(torch.from_numpy(g))
    st.cp_grad_sync()
    res = {"out": out.detach().numpy(), "dx": xt.grad.numpy()}
    for name, p in st.named_parameters():
        res["g_" + name] = p.grad.numpy()
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,lens,retain", [(2, [[9, 0, 30], [14, 3]], False), (3, [[21, 4], [], [8, 33]], True)])
def test_cp_stack_matches_single_device(tmp_path, world, lens, retain):
    mp.spawn(_worker, args=(world, _free_port(), lens, str(tmp_path), retain), nprocs=world, join=True)
    parts = [_batch(r, lens[r]) for r in range(world)]
    x = np.concatenate([p[0] for p in parts])
    ts = np.concatenate([p[1] for p in parts])
    g = np.concatenate([p[2] for p in parts])
    flat = [L for r in lens for L in r]
    offs = np.concatenate([[0], np.cumsum(flat)]).astype(np.int64)
    st = _stack()
    TorchOps.offsets_host = offs
    try:
        xt = torch.from_numpy(x).requires_grad_(True)
        out = st(xt, torch.from_numpy(ts), torch.from_numpy(offs), int(max(flat)))
        out.backward(torch.from_numpy(g))
    finally:
        TorchOps.offsets_host = None
    row = 0
    for r in range(world):
        res = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        n = parts[r][0].shape[0]
        np.testing.assert_allclose(res["out"], out.detach().numpy()[row:row + n], atol=1e-9, rtol=0)
        np.testing.assert_allclose(res["dx"], xt.grad.numpy()[row:row + n], atol=1e-9, rtol=0)
        for name, p in st.named_parameters():
            np.testing.assert_allclose(res["g_" + name], p.grad.numpy(), atol=1e-8, rtol=1e-9, err_msg=name)
        row += n


def test_layer_with_torch_ops_matches_oracle_attention():
    # the torch double's attention is the oracle's (pinned) forward
    rng = np.random.default_rng(0)
    lens = [5, 0, 17]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    q, k, v = (rng.standard_normal((T, H * DH)) for _ in range(3))
    ts = np.sort(rng.integers(0, 10**7, T))
    w = oracle.normal_init_ts_weights(16, 3)
    from _layer_ref import dense_attention
    got = dense_attention(*(torch.from_numpy(a) for a in (q, k, v, ts)), offs, torch.from_numpy(w), H, 16)
    want = oracle.hstu_forward(q, k, v, ts, offs, w, 16, H)
    np.testing.assert_allclose(got.numpy(), want, atol=1e-10)


def test_copy_params_roundtrip():
    a, b = _stack(), _stack()
    with torch.no_grad():
        for p in b.parameters():
            p.mul_(2)
    copy_params(a, b)
    for p1, p2 in zip(a.parameters(), b.parameters()):
        assert torch.equal(p1, p2)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_loopback_probe_runs_one_rank_share(k):
    # bench.py's CP max-length probe: one process = rank 0 of a CP group of k,
    # communication excluded; shapes / resident rows are exactly one rank's
    from paper_2508_04711_b200.cp_layer import CPAttention, LoopbackComm
    L = 64 * k
    cp = CPAttention(None, H, 16, backend=NumpyBackend(), comm=LoopbackComm(k, 0, peer_lengths=lambda r: []))
    st = _stack(cp)
    plan = cp.plan_for([L], torch.device("cpu"))
    n = plan[0].n_res
    assert n == L // k  # two balanced mini-chunks of L / (2k)
    x = torch.randn(n, E, dtype=torch.float64, requires_grad=True)
    ts = torch.cumsum(torch.randint(1, 1000, (n,)), 0)
    y = x
    for layer in st.layers:
        y = layer(y, ts, cp=(cp, plan))
    y.sum().backward()
    assert torch.isfinite(y).all() and torch.isfinite(x.grad).all()
