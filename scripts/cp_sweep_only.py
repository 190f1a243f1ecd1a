"""The bench's CP max-length sweep alone (GPU box)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

print(json.dumps(bench.cp_sweep(torch.device("cuda", 0), float(sys.argv[1]) if len(sys.argv) > 1 else 24.0)["rows"]))
