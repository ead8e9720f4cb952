"""Persistent kernels under a reduced SM budget (psk_set_sm_budget): grids
sized for a share of the GPU must give the same results (K1 CTA pairs with
an odd budget, K5 / K5-TC stream-K with fewer CTAs than blocks)."""

import pytest
import torch

from test_gemm_gpu import _gemm, _rand
from test_gemv_gpu import _run

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[37, 52])
def budget(request):
    from paper_2602_12029_b200 import _lib
    _lib.set_sm_budget(request.param)
    assert _lib.sm_budget() == request.param
    yield request.param
    _lib.set_sm_budget(0)
    assert _lib.sm_budget() == torch.cuda.get_device_properties(0).multi_processor_count


@pytest.mark.parametrize("M,N,K", [(4096, 6144, 4096), (300, 512, 256)])
def test_gemm_under_budget(budget, M, N, K):
    A, B = _rand(M, K, seed=41), _rand(N, K, std=0.02, seed=42)
    full = torch.empty(M, N, dtype=torch.float32, device="cuda")
    from paper_2602_12029_b200 import _lib
    _lib.set_sm_budget(0)
    _gemm(A, B, 1, full, N)
    _lib.set_sm_budget(budget)
    out = torch.empty_like(full)
    _gemm(A, B, 1, out, N)
    torch.cuda.synchronize()
    assert torch.equal(out, full)  # same k order per output whatever the grid


@pytest.mark.parametrize("rows,N", [([32, 32, 32, 32], 28672), ([16, 16], 4096), ([4, 4, 4, 4], 6144)])
def test_gemv_under_budget(budget, rows, N):
    _run(rows, N, 4096, 3 if N == 28672 else 2, seed=7, tc=max(rows) > 8)


def test_budget_rejects_bad_values():
    from paper_2602_12029_b200 import _lib
    with pytest.raises(_lib.PskError):
        _lib.set_sm_budget(-1)
    with pytest.raises(_lib.PskError):
        _lib.set_sm_budget(1)
