"""Multi-process (gloo, CPU) test of the SPMD jagged-CP layer's host logic.

The CP routing (plan, all-to-all redistribution, KV all-gather + sequence
re-order, dK/dV reduce-scatter to owners, restore) runs for real over
torch.distributed with world_size 2 and 3; the per-rank compute is injected as
a numpy backend (the GPU kernels are covered by the -m gpu tests).  Outputs
and gradients must equal the single-device oracle on the concatenated batch
(plan-independent, harness.py:171-186 reference_outputs).
"""

import math
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def _bias(tq, tk, w, nb):
    return np.asarray(w)[oracle.bucketize_array(tq[:, None] - tk[None, :], nb)]


class NumpyBackend:
    """Reference-semantics compute on CPU tensors (test double for GpuBackend)."""

    def gather(self, src, perm):
        return src.index_select(0, perm)

    def scatter(self, src, perm, out):
        out.index_copy_(0, perm, src)
        return out

    def _segs(self, segs):
        qo, qp, ks, kl = segs[:4]
        return qo.numpy(), qp.numpy(), ks.numpy(), kl.numpy()

    def fwd(self, q, k, v, ts_q, ts_k, segs, H, w, nb):
        qo, qp, ks, kl = self._segs(segs)
        Q, K, V = q.detach().numpy(), k.detach().numpy(), v.detach().numpy()
        tq, tk, w = ts_q.numpy(), ts_k.numpy(), w.detach().numpy()
        d = Q.shape[1] // H
        out = np.zeros_like(Q)
        for s in range(len(qp)):
            a, b = qo[s], qo[s + 1]
            kr = slice(ks[s], ks[s] + kl[s])
            mask = np.arange(kl[s])[None, :] <= (qp[s] + np.arange(b - a))[:, None]
            bias = _bias(tq[a:b], tk[kr], w, nb)
            for h in range(H):
                c = slice(h * d, (h + 1) * d)
                sc = (Q[a:b, c] @ K[kr, c].T + bias) / math.sqrt(d)
                out[a:b, c] = np.where(mask, oracle.silu(sc), 0.0) @ V[kr, c]
        return torch.from_numpy(out)

    def fwd_partial(self, q, k, v, ts_q, ts_k, segs, H, w, nb, acc, accumulate):
        out = self.fwd(q, k, v, ts_q, ts_k, segs, H, w, nb).to(acc.dtype)
        if accumulate:
            acc += out
        else:
            acc.copy_(out)

    def bwd_partial(self, q, k, v, ts_q, ts_k, segs, g, H, w, nb, dq_acc, dkv=None):
        dq, dk, dv, dw = self.bwd(q, k, v, ts_q, ts_k, segs, g, H, w, nb)
        dq_acc += dq
        if dkv is not None:
            dkv[0].add_(dk)
            dkv[1].add_(dv)
            return dkv[0], dkv[1], dw
        return dk, dv, dw

    def bwd(self, q, k, v, ts_q, ts_k, segs, g, H, w, nb):
        qo, qp, ks, kl = self._segs(segs)
        Q, K, V, G = q.detach().numpy(), k.detach().numpy(), v.detach().numpy(), g.detach().numpy()
        tq, tk, w = ts_q.numpy(), ts_k.numpy(), w.detach().numpy()
        d = Q.shape[1] // H
        dq, dk, dv = np.zeros_like(Q), np.zeros_like(K), np.zeros_like(V)
        dw = np.zeros(nb)
        for s in range(len(qp)):
            a, b = qo[s], qo[s + 1]
            kr = slice(ks[s], ks[s] + kl[s])
            mask = np.arange(kl[s])[None, :] <= (qp[s] + np.arange(b - a))[:, None]
            buckets = oracle.bucketize_array(tq[a:b, None] - tk[None, kr], nb)
            bias = w[buckets]
            for h in range(H):
                c = slice(h * d, (h + 1) * d)
                sc = (Q[a:b, c] @ K[kr, c].T + bias) / math.sqrt(d)
                sig = oracle.sigmoid(sc)
                A = np.where(mask, sc * sig, 0.0)
                dv[kr, c] += A.T @ G[a:b, c]
                dS = np.where(mask, (G[a:b, c] @ V[kr, c].T) * sig * (1 + sc * (1 - sig)), 0.0) / math.sqrt(d)
                dq[a:b, c] += dS @ K[kr, c]
                dk[kr, c] += dS.T @ Q[a:b, c]
                dw += np.bincount(buckets.ravel(), weights=dS.ravel(), minlength=nb)
        return (torch.from_numpy(dq), torch.from_numpy(dk), torch.from_numpy(dv), torch.from_numpy(dw))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _batch(seed, rank, lengths, D):
    rng = np.random.default_rng([seed, rank])
    T = int(sum(lengths))
    offs = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    q, k, v, g = (rng.standard_normal((T, D)) for _ in range(4))
    ts = np.zeros(T, dtype=np.int64)
    for b, L in enumerate(lengths):
        ts[offs[b]:offs[b] + L] = int(rng.integers(0, 10**9)) + np.cumsum(rng.integers(1, 10**6, size=L))
    return dict(q=q, k=k, v=v, g=g, ts=ts, offsets=offs)


def _worker(rank, world, port, lens, H, D, mode, result_dir, overlap=True, retain=False, protocol="alltoall"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04711_b200.cp_layer import CPAttention
    b = _batch(3, rank, lens[rank], H * D)
    w = torch.from_numpy(oracle.normal_init_ts_weights(16, 11))
    layer = CPAttention(dist.group.WORLD, H, 16, balance_mode=mode, backend=NumpyBackend(), overlap=overlap,
                        retain_kv=retain, protocol=protocol)
    t = {key: torch.from_numpy(b[key]) for key in ("q", "k", "v", "g", "ts")}
    out, ctx = layer.forward(t["q"], t["k"], t["v"], t["ts"], np.diff(b["offsets"]), w)
    dq, dk, dv, dw = layer.backward(ctx, t["g"], w)
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), out=out.numpy(), dq=dq.numpy(), dk=dk.numpy(),
             dv=dv.numpy(), dw=dw.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,lens,mode,overlap,retain,protocol", [
    (2, [[7, 0, 33], [12, 1]], "balanced_minichunk", True, False, "alltoall"),
    (2, [[7, 0, 33], [12, 1]], "balanced_minichunk", True, True, "allgather_split"),
    (2, [[7, 0, 33], [12, 1]], "balanced_minichunk", False, False, "alltoall"),
    (3, [[20, 5], [], [9, 40, 2]], "balanced_minichunk", True, False, "alltoall"),
    (3, [[20, 5], [], [9, 40, 2]], "balanced_minichunk", True, False, "allgather_split"),
    (2, [[31, 4], [17]], "naive_contiguous", True, True, "alltoall"),
])
def test_cp_layer_matches_single_device(tmp_path, world, lens, mode, overlap, retain, protocol):
    H, D = 2, 4
    mp.spawn(_worker, args=(world, _free_port(), lens, H, D, mode, str(tmp_path), overlap, retain, protocol),
             nprocs=world, join=True)
    batches = [_batch(3, r, lens[r], H * D) for r in range(world)]
    cat = oracle.concat_batches(batches)
    g = np.concatenate([b["g"] for b in batches])
    w = oracle.normal_init_ts_weights(16, 11)
    want = oracle.hstu_forward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], w, 16, H)
    wq, wk, wv, ww, _ = oracle.hstu_backward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], g, w, 16, H)
    row = 0
    for r in range(world):
        res = np.load(os.path.join(tmp_path, f"r{r}.npz"))
        n = batches[r]["q"].shape[0]
        sl = slice(row, row + n)
        for name, got, ref in (("out", res["out"], want[sl]), ("dq", res["dq"], wq[sl]), ("dk", res["dk"], wk[sl]),
                               ("dv", res["dv"], wv[sl])):
            assert got.shape == ref.shape and (got.size == 0 or np.abs(got - ref).max() < 1e-10), (r, name)
        assert np.abs(res["dw"] - ww).max() < 1e-10
        row += n


def _worker_steps(rank, world, port, steps, H, D, result_dir, staged, prefetch=False):
    """Variable batches over several steps: some ranks repeat their local
    lengths while others change (the plan-cache divergence scenario)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_04711_b200.cp_layer import CPAttention, HostStagedComm
    w = torch.from_numpy(oracle.normal_init_ts_weights(16, 11))
    comm = HostStagedComm(dist.group.WORLD) if staged else None
    layer = CPAttention(dist.group.WORLD, H, 16, backend=NumpyBackend(), comm=comm, max_plans=2)
    res = {}
    for i, lens in enumerate(steps):
        b = _batch(10 + i, rank, lens[rank], H * D)
        t = {key: torch.from_numpy(b[key]) for key in ("q", "k", "v", "g", "ts")}
        out, ctx = layer.forward(t["q"], t["k"], t["v"], t["ts"], np.diff(b["offsets"]), w)
        if prefetch and i + 1 < len(steps):  # next step's length exchange, started before this backward
            layer.prefetch_plan(steps[i + 1][rank])
        dq, dk, dv, dw = layer.backward(ctx, t["g"], w)
        res[f"out{i}"], res[f"dq{i}"], res[f"dw{i}"] = out.numpy(), dq.numpy(), dw.numpy()
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("staged,prefetch", [(False, False), (True, False), (False, True)])
def test_cp_plan_cache_consistent_across_variable_batches(tmp_path, staged, prefetch):
    world, H, D = 2, 1, 4
    steps = [[[7, 3], [12]], [[7, 3], [5, 9]], [[4], [5, 9]], [[7, 3], [12]], [[7, 3], [5, 9]]]
    mp.spawn(_worker_steps, args=(world, _free_port(), steps, H, D, str(tmp_path), staged, prefetch), nprocs=world,
             join=True)
    w = oracle.normal_init_ts_weights(16, 11)
    res = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    for i, lens in enumerate(steps):
        batches = [_batch(10 + i, r, lens[r], H * D) for r in range(world)]
        cat = oracle.concat_batches(batches)
        g = np.concatenate([b["g"] for b in batches])
        want = oracle.hstu_forward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], w, 16, H)
        wq, _, _, ww, _ = oracle.hstu_backward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], g, w, 16, H)
        row = 0
        for r in range(world):
            n = batches[r]["q"].shape[0]
            assert np.abs(res[r][f"out{i}"] - want[row:row + n]).max(initial=0) < 1e-10, (i, r)
            assert np.abs(res[r][f"dq{i}"] - wq[row:row + n]).max(initial=0) < 1e-10, (i, r)
            assert np.abs(res[r][f"dw{i}"] - ww).max() < 1e-10, (i, r)
            row += n


def _worker_cpdp(rank, world, port, cp, lens, H, D, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2508_04711_b200.cp_layer import CPJaggedHSTUAttention, make_cp_dp_groups
    cp_group, dp_group, ci, di = make_cp_dp_groups(cp)
    w = oracle.normal_init_ts_weights(16, 11)
    mod = CPJaggedHSTUAttention(cp_group, H, 16, backend=NumpyBackend(), weights=w)
    model = DDP(mod, process_group=dp_group)
    b = _batch(3, rank, lens[rank], H * D)
    t = {key: torch.from_numpy(b[key]) for key in ("q", "k", "v", "g", "ts")}
    for key in ("q", "k", "v"):
        t[key].requires_grad_(True)
    out = model(t["q"], t["k"], t["v"], t["ts"], np.diff(b["offsets"]))
    (out * t["g"]).sum().backward()
    np.savez(os.path.join(result_dir, f"r{rank}.npz"), out=out.detach().numpy(), dq=t["q"].grad.numpy(),
             dk=t["k"].grad.numpy(), dv=t["v"].grad.numpy(), dw=mod.ts_weights.grad.numpy(), ci=ci, di=di)
    dist.destroy_process_group()


def test_hybrid_cp_dp_gradient_semantics(tmp_path):
    """CP2 x DP2 (config C5's layout at world 4): outputs / input gradients
    equal the single-device oracle on each CP group's batch; the ts_weights
    gradient is the SUM over CP and the MEAN over DP (DDP over the DP group)."""
    world, cp, H, D = 4, 2, 1, 4
    lens = [[9, 0, 20], [13], [5, 30], [8, 8]]
    mp.spawn(_worker_cpdp, args=(world, _free_port(), cp, lens, H, D, str(tmp_path)), nprocs=world, join=True)
    w = oracle.normal_init_ts_weights(16, 11).astype(np.float32).astype(np.float64)
    dws = []
    res = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    for grp in range(world // cp):
        ranks = list(range(grp * cp, (grp + 1) * cp))
        batches = [_batch(3, r, lens[r], H * D) for r in ranks]
        cat = oracle.concat_batches(batches)
        g = np.concatenate([b["g"] for b in batches])
        want = oracle.hstu_forward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], w, 16, H)
        wq, wk, wv, ww, _ = oracle.hstu_backward(cat["q"], cat["k"], cat["v"], cat["ts"], cat["offsets"], g, w, 16, H)
        dws.append(ww)
        row = 0
        for r in ranks:
            assert int(res[r]["ci"]) == r % cp and int(res[r]["di"]) == grp
            n = batches[r - ranks[0]]["q"].shape[0]
            for name, ref in (("out", want), ("dq", wq), ("dk", wk), ("dv", wv)):
                assert np.abs(res[r][name] - ref[row:row + n]).max(initial=0) < 1e-9, (r, name)
            row += n
    expect = np.mean(dws, axis=0)
    for r in range(world):
        assert np.abs(res[r]["dw"] - expect).max() < 1e-6 * max(1.0, np.abs(expect).max()), r
