"""Hardware pin of the tcgen05 descriptor encodings (GPU)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("a_mode,b_mode", [(0, 0), (0, 1), (1, 1), (2, 1), (2, 0), (3, 0), (4, 1), (1, 0)])
def test_umma_tile(a_mode, b_mode):
    from paper_2508_04711_b200 import kernels
    g = torch.Generator().manual_seed(a_mode * 10 + b_mode)
    A = torch.randn(128, 128, generator=g).bfloat16()
    B = torch.randn(128, 128, generator=g).bfloat16()
    a_store = A if a_mode in (0, 2, 3) else A.t().contiguous()
    b_store = B.t().contiguous() if b_mode == 0 else B
    d = kernels.debug_umma(a_store.cuda(), b_store.cuda(), a_mode, b_mode)
    torch.cuda.synchronize()
    want = A.float() @ B.float()
    err = (d.cpu() - want).abs().max().item()
    assert err < 1e-2, f"a_mode={a_mode} b_mode={b_mode} max err {err}"
