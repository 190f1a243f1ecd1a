"""Bisect helper: blockwise_partial on random key partitions (GPU box)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from _cases import make_case  # noqa: E402
import paper_2508_04711_b200 as pkg  # noqa: E402
from paper_2508_04711_b200 import attention  # noqa: E402

lens = [int(x) for x in sys.argv[1].split(",")]
d = int(sys.argv[2])
frac = float(sys.argv[3])
case = make_case(lens, d, seed=1)
offs = case["offsets"]
seq = np.repeat(np.arange(len(lens)), lens)
pos = np.concatenate([np.arange(L) for L in lens])
idx = np.sort(np.random.default_rng(1).permutation(int(offs[-1]))[: max(1, int(frac * offs[-1]))])
segs = attention._blockwise_segments(seq, pos, seq[idx], pos[idx])
print("nseg", segs[2].size - 1, "pos0 max", segs[3].max(), "kvl", segs[5].min(), segs[5].max(), flush=True)
t0 = time.time()
out = pkg.blockwise_partial(case["q"], seq, pos, case["ts"], case["k"][idx], seq[idx], pos[idx], case["ts"][idx],
                            case["v"][idx], pkg.BiasParams(case["w"]), pkg.BiasConfig(16))
torch.cuda.synchronize()
print("ok", time.time() - t0, float(out.abs().sum()), flush=True)
