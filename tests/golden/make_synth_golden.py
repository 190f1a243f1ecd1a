"""Freeze the reference generator's integer stream (harness.py:123-145):
offsets and timestamps of ``gen_synthetic_batch`` for a few seeded configs,
in both draw dtypes, from the UNMODIFIED reference (build container only):

    python tests/golden/make_synth_golden.py

``tests/test_boundary_cpu.py`` checks ``harness.gen_synthetic_host`` against
them bit for bit (the bf16 tag draws the reference's f64 stream)."""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from jaggedcp import harness  # noqa: E402
    cases = []
    for seed, dist, dtype, bs, max_len, max_length in ((7, "uniform", "f64", 6, 300, 1024),
                                                       (7, "uniform", "f32", 6, 300, 1024),
                                                       (3, "lognormal", "f64", 5, 0, 8192),
                                                       (23, "uniform", "f64", 2, 24, 32)):
        kw = dict(cp_size=2, batch_size=bs, length_dist=dist, max_length=max_length, embed_dim=8, dtype=dtype,
                  seed=seed)
        if dist == "uniform":
            kw.update(min_len=0, max_len=max_len)
        else:
            kw.update(lognorm_mu=float(np.log(1024)), lognorm_sigma=1.0)
        cfg = harness.ExperimentConfig(**kw)
        for rank in range(2):
            b = harness.gen_synthetic_batch(cfg, rank)
            cases.append({"cfg": kw, "rank": rank, "offsets": [int(x) for x in b.q.offsets],
                          "ts": [int(x) for x in b.ts.values],
                          "q_sum": float(np.asarray(b.q.values, dtype=np.float64).sum())})
    with open(os.path.join(HERE, "synthetic.json"), "w") as f:
        json.dump(cases, f)
    print("wrote", os.path.join(HERE, "synthetic.json"))


if __name__ == "__main__":
    main()
