"""Achieved HBM bandwidth of the bandwidth-bound helpers (SURVEY §8(d) byte
formulas) on C2-scale and larger inputs, against MEASURED_PEAKS.json hbm_gbs.

    python scripts/bench_helpers.py [out.json]

Each helper runs on inputs larger than L2 (or is timed after an L2 flush),
warm-up 3, then the median of 10 launches timed with CUDA events on the
launching stream.  Bytes are algorithmic (what the helper must read + write).
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_04711_b200 import kernels  # noqa: E402


def timed(fn, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts))


def main():
    dev = "cuda"
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    rng = np.random.default_rng(0)
    rows = []

    def rec(name, sec, nbytes, shape):
        rows.append({"helper": name, "shape": shape, "bytes": int(nbytes), "us": sec * 1e6,
                     "GB_s": nbytes / sec / 1e9, "frac_hbm": nbytes / sec / 1e9 / peak})

    # jagged <-> padded: 8x the C2 batch (B=256, L<=1024, 512 bf16 columns)
    lens = rng.integers(1, 1025, size=256)
    offs = torch.from_numpy(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)).to(dev)
    T, B, L, D = int(lens.sum()), len(lens), 1024, 512
    vals = torch.randn(T, D, device=dev).bfloat16()
    padded = kernels.jagged_to_padded(vals, offs, L)
    rec("jagged_to_padded", timed(lambda: kernels.jagged_to_padded(vals, offs, L), flush),
        T * D * 2 + B * L * D * 2, [T, D])
    rec("padded_to_jagged", timed(lambda: kernels.padded_to_jagged(padded, offs, T), flush), 2 * T * D * 2, [B, L, D])
    # row gather / scatter (CP pack / reorder), 2 * rows * row_bytes
    perm = torch.from_numpy(rng.permutation(T).astype(np.int64)).to(dev)
    out = torch.empty_like(vals)
    rec("gather_rows", timed(lambda: kernels.gather_rows(vals, perm, out), flush), 2 * T * D * 2, [T, D])
    rec("scatter_rows", timed(lambda: kernels.scatter_rows(vals, perm, out), flush), 2 * T * D * 2, [T, D])
    # bucketize: int64 deltas in, int32 buckets out
    n = 64 * 1024 * 1024
    deltas = torch.randint(-10, 10**7, (n,), device=dev, dtype=torch.int64)
    rec("bucketize", timed(lambda: kernels.bucketize(deltas, 16), flush), n * (8 + 4), [n])
    # compute_bias (one 8192^2 block): sum L^2 * 4 written + 2 L * 8 read
    Lb = 8192
    ts = torch.cumsum(torch.randint(1, 10**6, (Lb,), device=dev), 0)
    w = torch.randn(16, device=dev) * 0.02
    bias = kernels.compute_bias(ts, ts, w, 16)
    rec("compute_bias", timed(lambda: kernels.compute_bias(ts, ts, w, 16), flush), Lb * Lb * 4 + 2 * Lb * 8, [Lb, Lb])
    # d_ts_weights scatter from a materialised dBias: sum L^2 * 4 read
    dw = torch.zeros(16, dtype=torch.float64, device=dev)
    rec("dbias_scatter", timed(lambda: kernels.dbias_scatter(ts, ts, bias, 16, dw), flush), Lb * Lb * 4 + 2 * Lb * 8,
        [Lb, Lb])
    # HSTU layer row kernels at the C4 batch scale x4 (180K rows): silu over uvqk
    # (4 H d = 2048 columns, read + write), norm_gate over the attention output
    # (512 columns, gate = strided u view): fwd reads x, u, writes y (+ 8 B stats),
    # bwd reads dy, x, u, writes dx, du
    R, N = 180_420, 512
    uvqk = torch.randn(R, 4 * N, device=dev).bfloat16()
    rec("silu_fwd", timed(lambda: kernels.silu(uvqk), flush), 2 * R * 4 * N * 2, [R, 4 * N])
    dyu = torch.randn(R, 4 * N, device=dev).bfloat16()
    rec("silu_bwd", timed(lambda: kernels.silu_bwd(uvqk, dyu), flush), 3 * R * 4 * N * 2, [R, 4 * N])
    # + the uvqk bias gradient in the same pass (partial rows + column sweep included)
    rec("silu_bwd_colsum", timed(lambda: kernels.silu_bwd_colsum(uvqk, dyu), flush), 3 * R * 4 * N * 2,
        [R, 4 * N])
    dyn = dyu[:, :N].contiguous()
    rec("colsum", timed(lambda: kernels.colsum(dyn), flush), R * N * 2, [R, N])
    xa = torch.randn(R, N, device=dev).bfloat16()
    u = uvqk[:, :N]
    g_, b_ = torch.ones(N, device=dev), torch.zeros(N, device=dev)
    y, mean, rstd = kernels.norm_gate_fwd(xa, u, g_, b_)
    rec("norm_gate_fwd", timed(lambda: kernels.norm_gate_fwd(xa, u, g_, b_), flush), 3 * R * N * 2 + 8 * R, [R, N])
    dy = torch.randn(R, N, device=dev).bfloat16()
    rec("norm_gate_bwd", timed(lambda: kernels.norm_gate_bwd(dy, xa, u, g_, b_, mean, rstd), flush),
        5 * R * N * 2 + 8 * R, [R, N])
    res = {"peak_hbm_gbs": peak, "peak_kind": "MEASURED_PEAKS.json copy bandwidth", "rows": rows,
           "device": torch.cuda.get_device_name()}
    for r in rows:
        print(f"{r['helper']:18s} {r['us']:9.1f} us  {r['GB_s']:8.0f} GB/s  {r['frac_hbm']:.2f} of HBM")
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
