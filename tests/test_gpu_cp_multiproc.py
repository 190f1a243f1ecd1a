"""The CUDA CP layer (cp_layer.CPAttention with the real GpuBackend kernels)
at world size 2 and 4: several processes share cuda:0 and exchange through a
gloo group staged in host memory (cp_layer.HostStagedComm).  No kernel waits
on another process (the exchange is host-side), so sharing one GPU is safe.

Outputs and gradients (out, dq, dk, dv, d_ts_weights) must match the CPU
oracle on the concatenated batch (harness.py:171-186: CP results are
plan-independent), for C3-shaped (uniform) and skewed (lognormal) lengths, in
both balance modes, overlapped and not.  Tolerance: row-normalised error
(harness.py:189-206) <= ROW_TOL for bf16 inputs; d_w <= 1e-3 of max |d_w|.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from _cases import bf16_round, row_rel

pytestmark = pytest.mark.gpu

ROW_TOL = 1e-2  # lengths up to 2048 and fp32 CP partial sums: 4-6.5e-3 measured
H, d = 2, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _batch(seed, rank, dist_kind, B):
    rng = np.random.default_rng([seed, rank])
    if dist_kind == "uniform":
        lens = rng.integers(1, 1537, size=B)
    else:
        lens = np.clip(np.floor(rng.lognormal(np.log(256), 1.0, size=B)), 1, 2048).astype(np.int64)
    lens[0] = 0 if rank == 1 else lens[0]  # an empty sequence on one rank
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    T = int(offs[-1])
    q, k, v, g = (bf16_round(rng.standard_normal((T, H * d)).astype(np.float32)) for _ in range(4))
    ts = np.zeros(T, dtype=np.int64)
    for b, L in enumerate(lens):
        ts[offs[b]:offs[b] + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, 10**6 + 1, size=L))
    return dict(q=q, k=k, v=v, g=g, ts=ts, offsets=offs)


def _worker(rank, world, port, dist_kind, B, mode, overlap, out_dir, protocol="alltoall", retain=False,
            budget=None):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if budget:  # a dS budget below the calls' whole-segment scratch: the windowed backward
        os.environ["JH_DS_SCRATCH_BUDGET"] = budget
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04711_b200.cp_layer import CPAttention, HostStagedComm
    b = _batch(17, rank, dist_kind, B)
    w = torch.from_numpy(oracle.normal_init_ts_weights(16, 23).astype(np.float32)).cuda()
    layer = CPAttention(dist.group.WORLD, H, 16, balance_mode=mode, overlap=overlap,
                        comm=HostStagedComm(dist.group.WORLD), protocol=protocol, retain_kv=retain)
    t = {x: torch.from_numpy(b[x]).cuda().bfloat16() for x in ("q", "k", "v", "g")}
    ts = torch.from_numpy(b["ts"]).cuda()
    lens = np.diff(b["offsets"])
    for _ in range(2):  # second step: the cached plan path
        out, ctx = layer.forward(t["q"], t["k"], t["v"], ts, lens, w)
        dq, dk, dv, dw = layer.backward(ctx, t["g"], w)
    torch.cuda.synchronize()
    if budget:
        from paper_2508_04711_b200 import kernels
        assert kernels.WINDOWED_BWD["calls"] > 0, "the windowed backward did not run"
    f = lambda x: x.float().cpu().numpy()  # noqa: E731
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), out=f(out), dq=f(dq), dk=f(dk), dv=f(dv),
             dw=dw.double().cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dist_kind,B,mode,overlap,protocol,retain,budget", [
    (2, "uniform", 3, "balanced_minichunk", True, "alltoall", False, None),
    (2, "uniform", 3, "naive_contiguous", False, "alltoall", False, None),
    (2, "uniform", 3, "balanced_minichunk", True, "allgather_split", True, None),
    (4, "lognormal", 3, "balanced_minichunk", True, "alltoall", False, None),
    (4, "lognormal", 2, "naive_contiguous", True, "allgather_split", False, None),
    (2, "uniform", 3, "balanced_minichunk", True, "alltoall", False, "2e6"),
    (2, "uniform", 3, "naive_contiguous", True, "alltoall", True, "2e6"),
])
def test_cuda_cp_layer_matches_oracle(tmp_path, world, dist_kind, B, mode, overlap, protocol, retain, budget):
    mp.spawn(_worker, args=(world, _free_port(), dist_kind, B, mode, overlap, str(tmp_path), protocol, retain,
                            budget),
             nprocs=world, join=True)
    batches = [_batch(17, r, dist_kind, B) for r in range(world)]
    cat = oracle.concat_batches(batches)
    g = np.concatenate([b["g"] for b in batches])
    w = oracle.normal_init_ts_weights(16, 23).astype(np.float32).astype(np.float64)
    want = oracle.hstu_forward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], w, 16, H)
    wq, wk, wv, ww, _ = oracle.hstu_backward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], g, w, 16, H)
    row = 0
    for r in range(world):
        res = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        n = batches[r]["q"].shape[0]
        for name, ref in (("out", want), ("dq", wq), ("dk", wk), ("dv", wv)):
            mx, rel = row_rel(res[name], ref[row:row + n]) if n else (0.0, 0.0)
            print(f"world={world} rank={r} {name}: max_abs={mx:.3e} row_rel={rel:.3e}")
            assert rel <= ROW_TOL, (r, name, rel)
        err = np.abs(res["dw"] - ww).max() / np.abs(ww).max()
        print(f"world={world} rank={r} d_w rel-to-max={err:.3e}")
        assert err <= 1e-3
        row += n


# ------------------------------------- CP-sharded HSTU stack on the CUDA kernels

def _stack_inputs(rank, lens, E):
    rng = np.random.default_rng([41, rank])
    T = int(sum(lens))
    x = rng.standard_normal((T, E)).astype(np.float32)
    ts = np.zeros(T, dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    for b, L in enumerate(lens):
        ts[offs[b]:offs[b] + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, 10**6, size=L))
    gy = rng.standard_normal((T, E)).astype(np.float32)
    return x, ts, gy


def _stack_worker(rank, world, port, lens, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04711_b200.cp_layer import CPAttention, HostStagedComm
    from paper_2508_04711_b200.hstu_layer import HSTUStack
    E, Hh, dh = 256, 2, 128
    cp = CPAttention(dist.group.WORLD, Hh, 16, comm=HostStagedComm(dist.group.WORLD))
    st = HSTUStack(2, E, Hh, dh, 16, seed=3, cp=cp).cuda()
    x, ts, gy = _stack_inputs(rank, lens[rank], E)
    xt = torch.from_numpy(x).cuda().bfloat16().requires_grad_(True)
    out = st(xt, torch.from_numpy(ts).cuda(), local_lengths=lens[rank])
    out.backward(torch.from_numpy(gy).cuda().bfloat16())
    st.cp_grad_sync()
    torch.cuda.synchronize()
    res = {"out": out.detach().float().cpu().numpy(), "dx": xt.grad.float().cpu().numpy()}
    for name, p in st.named_parameters():
        res["g_" + name] = p.grad.float().cpu().numpy()
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), **res)
    dist.destroy_process_group()


def test_cuda_cp_stack_world2_matches_single_process(tmp_path):
    # activations CP-sharded across 2 layers, K/V exchanged per layer, the
    # CP x DP gradient rule (cp_grad_sync): equal to the plain stack on the
    # concatenated batch up to bf16 rounding
    from paper_2508_04711_b200.hstu_layer import HSTUStack
    world, E = 2, 256
    lens = [[700, 1, 300], [129, 900]]
    mp.spawn(_stack_worker, args=(world, _free_port(), lens, str(tmp_path)), nprocs=world, join=True)
    parts = [_stack_inputs(r, lens[r], E) for r in range(world)]
    x = np.concatenate([p[0] for p in parts])
    ts = np.concatenate([p[1] for p in parts])
    gy = np.concatenate([p[2] for p in parts])
    flat = [L for r in lens for L in r]
    offs = np.concatenate([[0], np.cumsum(flat)]).astype(np.int64)
    st = HSTUStack(2, E, 2, 128, 16, seed=3).cuda()
    xt = torch.from_numpy(x).cuda().bfloat16().requires_grad_(True)
    out = st(xt, torch.from_numpy(ts).cuda(), torch.from_numpy(offs).cuda(), max(flat))
    out.backward(torch.from_numpy(gy).cuda().bfloat16())
    torch.cuda.synchronize()
    row = 0
    for r in range(world):
        res = np.load(os.path.join(tmp_path, f"s{r}.npz"))
        n = parts[r][0].shape[0]
        e_out = row_rel(res["out"], out.detach().float().cpu().numpy()[row:row + n])[1]
        e_dx = row_rel(res["dx"], xt.grad.float().cpu().numpy()[row:row + n])[1]
        print(f"rank {r}: out {e_out:.2e} dx {e_dx:.2e}")
        assert e_out <= 2e-2 and e_dx <= 2e-2
        for name, p in st.named_parameters():
            ref = p.grad.float().cpu().numpy()
            e = np.abs(res["g_" + name] - ref).max() / max(np.abs(ref).max(), 1e-6)
            assert e <= 3e-2, (r, name, e)
        row += n
