"""Debug helper: run one fused forward/backward config in this process."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from _cases import make_case, to_cuda, row_rel
import oracle
from paper_2508_04711_b200 import kernels
lens = [int(x) for x in sys.argv[1].split(",")]
H, d = int(sys.argv[2]), int(sys.argv[3])
which = sys.argv[4] if len(sys.argv) > 4 else "fwd"
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 1
case = make_case(lens, H * d, seed=seed)
c = to_cuda(case)
try:
    if which == "fwd":
        out = kernels.attn_fwd(c["q"], c["k"], c["v"], c["ts"], c["ts"], c["offsets"], H, c["w"], 16)
        torch.cuda.synchronize()
        want = oracle.hstu_forward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["w"], 16, H)
        print(lens, H, d, which, "rel", row_rel(out.float().cpu().numpy(), want))
    else:
        dq, dk, dv, dw, _ = kernels.attn_bwd(c["q"], c["k"], c["v"], c["ts"], c["ts"], c["offsets"], c["g"], H, c["w"], 16)
        torch.cuda.synchronize()
        wq, wk, wv, ww, _ = oracle.hstu_backward(case["q"], case["k"], case["v"], case["ts"], case["offsets"], case["g"], case["w"], 16, H)
        dwe = float(np.abs(dw.cpu().numpy() - ww).max() / np.abs(ww).max())
        print(lens, H, d, which, "rel", [row_rel(a.float().cpu().numpy(), b)[1] for a, b in ((dq, wq), (dk, wk), (dv, wv))], "dw", dwe)
except Exception as e:
    print(lens, H, d, which, "ERROR", str(e).splitlines()[0])
