import sys, json, torch
sys.path.insert(0, '.')
from paper_2508_04711_b200 import kernels
from paper_2508_04711_b200.harness import sweep_max_tokens_measured
for en in (True, False):
    kernels.WINDOWED_BWD["enabled"] = en
    rep = sweep_max_tokens_measured(int(24e9), (8,), embed_dim=512, num_heads=4, num_layers=8, num_buckets=16, seed=7,
                                    device=torch.device("cuda", 0), time_budget_s=400)
    print("windowed", en, json.dumps(rep.rows), flush=True)
