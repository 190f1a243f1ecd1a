"""Freeze the reference's memory-budget length sweep (harness.py:319-368,
``modeled_rank_bytes`` / ``sweep_max_tokens``) and the key set of its
``ExperimentReport`` JSON (harness.py:213-253) into ``sweep.json``.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_sweep_golden.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from jaggedcp import harness  # noqa: E402


def main():
    rec = {"sweeps": [], "modeled": [], "report_keys": None}
    for budget, cps, dim, dt in ((16_777_216, [1, 2, 4, 8], 8, "f32"), (1 << 30, [1, 2, 4, 8, 16], 512, "f32"),
                                 (80 << 30, [1, 4, 8], 512, "f64")):
        rep = harness.sweep_max_tokens(budget, cps, embed_dim=dim, dtype=dt)
        rec["sweeps"].append({"budget": budget, "cp_sizes": cps, "embed_dim": dim, "dtype": dt,
                              "json": rep.to_json_dict()})
    for L in (1, 7, 100, 4096, 16384, 100_003):
        for cp in (1, 2, 3, 4, 8):
            rec["modeled"].append({"L": L, "cp": cp, "embed_dim": 8, "dtype_size": 4,
                                   "bytes": harness.modeled_rank_bytes(L, cp, 8, 4)})
    cfg = harness.ExperimentConfig(cp_size=2, batch_size=2, min_len=0, max_len=24, max_length=32, seed=23)
    payload = harness.run_experiment(cfg).to_json_dict()
    rec["report_keys"] = {k: sorted(v.keys()) if isinstance(v, dict) else None for k, v in payload.items()}
    with open(os.path.join(HERE, "sweep.json"), "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "sweep.json"))


if __name__ == "__main__":
    main()
