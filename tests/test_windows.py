"""CPU check of the windowed backward's decomposition (kernels.window_segments):
every visible (q row, kv row) pair of a segment-form call -- kv position j of
segment s visible to q row i iff j < kv_len[s] and j <= q_pos0[s] + i -- is
covered by exactly one window call, with the compact kv copy mapping back to
the original kv rows.  Plain self-attention and CP-like segment layouts."""

import numpy as np
import pytest

from paper_2508_04711_b200 import kernels


def _pairs_original(qo, qp, kl, ks):
    out = []
    for s in range(qp.size):
        for i in range(int(qo[s + 1] - qo[s])):
            for j in range(int(kl[s])):
                if j <= qp[s] + i:
                    out.append((int(qo[s] + i), int(ks[s] + j)))
    return sorted(out)


def _pairs_windows(wins):
    out = []
    for o_a, qp_a, kl_a, host, c in wins:
        m = qp_a.size
        ks_a = host[2 * m + 1:3 * m + 1]
        rows = host[4 * m + 1:]
        assert rows.size == c
        for t in range(m):
            for r in range(int(o_a[t]), int(o_a[t + 1])):
                for j in range(int(kl_a[t])):
                    if j <= qp_a[t] + (r - o_a[t]):
                        out.append((r, int(rows[ks_a[t] + j])))
    return sorted(out)


@pytest.mark.parametrize("W,chunk", [(128, 16384), (128, 96), (256, 200), (384, 1024)])
def test_plain_self_attention(W, chunk):
    lens = np.array([300, 0, 1, 700, 129])
    qo = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    segs = (qo, np.zeros(lens.size, np.int64), lens.astype(np.int64), qo[:-1].copy())
    wins = kernels.window_segments(segs, W, chunk)
    assert _pairs_windows(wins) == _pairs_original(*segs)
    assert all(np.all(w[2] <= W) for w in wins)  # no window is wider than W


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_segment_form(seed):
    # CP-like: q rows at positions q_pos0 + i against kv prefixes / gaps of another layout
    rng = np.random.default_rng(seed)
    nseg = 6
    qlen = rng.integers(0, 300, nseg)
    qo = np.concatenate([[0], np.cumsum(qlen)]).astype(np.int64)
    qp = rng.integers(0, 600, nseg).astype(np.int64)
    kl = rng.integers(0, 700, nseg).astype(np.int64)
    ks = rng.integers(0, 2000, nseg).astype(np.int64)
    segs = (qo, qp, kl, ks)
    for W, chunk in ((128, 64), (256, 1000)):
        assert _pairs_windows(kernels.window_segments(segs, W, chunk)) == _pairs_original(*segs)
