"""K5 grouped decode GEMV (TMA-bulk weight stream + mma.sync, 1..32 rows per
module) and K5-TC (tcgen05, 9..64 rows per module) vs a torch fp32 reference on identical bf16 operands, all
epilogues, ragged rows per module (incl. modules with no rows, one module
holding every row, K not a multiple of the 1024-column stage).
Tolerance: |gpu - ref| <= 2e-3 * max|ref| + 1e-4 (fp32 outputs),
1e-2 * max|ref| + 1e-3 (bf16 outputs)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(rows_per_mod, N, K, epi, seed=0, tc=False):
    import ctypes
    from paper_2602_12029_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_mod = len(rows_per_mod)
    W = [(torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16) for _ in range(n_mod)]
    R = sum(rows_per_mod)
    x = torch.randn(R, K, device="cuda", generator=g).to(torch.bfloat16)
    mrs = [0]
    for r in rows_per_mod:
        mrs.append(mrs[-1] + r)
    ptrs = torch.tensor([w.data_ptr() for w in W], dtype=torch.int64, device="cuda")
    t_mrs = torch.tensor(mrs, dtype=torch.int32, device="cuda")
    ref = torch.zeros(R, N, device="cuda")
    for i in range(n_mod):
        ref[mrs[i]:mrs[i + 1]] = x[mrs[i]:mrs[i + 1]].float() @ W[i].float().T
    if epi == 3:
        y = ref.view(R, -1, 2, 8)
        ref = (torch.nn.functional.silu(y[:, :, 0]) * y[:, :, 1]).reshape(R, N // 2)
        out = torch.zeros(R, N // 2, dtype=torch.bfloat16, device="cuda")
    elif epi == 0:
        out = torch.zeros(R, N, dtype=torch.bfloat16, device="cuda")
    else:
        out = torch.randn(R, N, device="cuda", generator=g) if epi == 2 else torch.zeros(R, N, device="cuda")
        if epi == 2:
            ref = ref + out
    lib = _lib.load()
    if tc:
        hp = (ctypes.c_void_p * n_mod)(*[w.data_ptr() for w in W])
        wsb = ctypes.c_int64()
        _lib.check(lib.psk_gemv_tc_workspace(ctypes.byref(wsb)))
        ws = torch.zeros(wsb.value, dtype=torch.uint8, device="cuda")
        for _ in range(2):  # twice: the stream-K flags must come back zeroed
            o2 = out.clone()
            _lib.check(lib.psk_gemv_tc(x.data_ptr(), R, K, hp, t_mrs.data_ptr(), n_mod, max(rows_per_mod), N,
                                       epi, o2.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream))
        assert int(ws[:4096].view(torch.int32).abs().sum().item()) == 0
        out = o2
    else:
        _lib.check(lib.psk_gemv(x.data_ptr(), R, K, ptrs.data_ptr(), t_mrs.data_ptr(), n_mod, max(rows_per_mod), N,
                                epi, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    tol = (1e-2 * scale + 1e-3) if epi in (0, 3) else (2e-3 * scale + 1e-4)
    assert err <= tol, f"err {err} scale {scale}"


@pytest.mark.parametrize("rows", [[1, 1, 1, 1], [2, 2], [4, 4, 4, 4], [8, 3, 0, 5], [16, 16], [12, 1], [0, 0, 16, 0],
                                  [32, 5], [0, 17]])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_gemv_rows_and_epilogues(rows, epi):
    _run(rows, 1536, 4096, epi)


@pytest.mark.parametrize("N,K", [(256, 768), (4096, 14336), (6144, 4096)])
def test_gemv_shapes(N, K):
    _run([3, 5, 2, 6], N, K, 1, seed=1)
    _run([1, 1, 1], N, K, 1, seed=2)


@pytest.mark.parametrize("N,K", [(48, 1160), (128256 // 8, 4096)])
def test_gemv_ragged_k_and_many_tiles(N, K):
    """K = 1160: a partial last stage (136 columns, not a multiple of 32);
    N = 16032: more tiles than SMs per module."""
    _run([2, 1], N, K, 1, seed=3)
    _run([5], N, K, 2, seed=4)


@pytest.mark.parametrize("rows", [[9, 16, 3, 16], [32, 5], [0, 17], [64, 64, 1, 40], [33], [0, 0, 48, 0],
                                  [16] * 8, [20] * 16])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_gemv_tc_rows_and_epilogues(rows, epi):
    _run(rows, 1536, 4096, epi, tc=True)


@pytest.mark.parametrize("N,K", [(4096, 14336), (6144, 4096), (16384, 4096), (128, 64), (28672, 4096)])
def test_gemv_tc_shapes(N, K):
    _run([30, 31, 2, 16], N, K, 1, seed=1, tc=True)
    _run([12], N, K, 2, seed=2, tc=True)
    _run([16, 9, 0, 3], N, K, 3 if N % 16 == 0 else 1, seed=3, tc=True)   # <= 16 rows: two-block units at N >= 16384


@pytest.mark.parametrize("rows,N,K,epi", [([32, 32, 32, 32], 4096, 4096, 2), ([16, 16, 16, 16], 28672, 4096, 3),
                                          ([64, 5], 6144, 4096, 1)])
def test_gemv_tc_bit_reproducible(rows, N, K, epi):
    """Stream-K blocks split between CTAs are reduced in a fixed order: two
    launches give bit-identical outputs."""
    import ctypes
    from paper_2602_12029_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(5)
    W = [(torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16) for _ in rows]
    R = sum(rows)
    x = torch.randn(R, K, device="cuda", generator=g).to(torch.bfloat16)
    mrs = torch.tensor([0] + list(np.cumsum(rows)), dtype=torch.int32, device="cuda")
    hp = (ctypes.c_void_p * len(rows))(*[w.data_ptr() for w in W])
    wsb = ctypes.c_int64()
    _lib.check(_lib.load().psk_gemv_tc_workspace(ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value, dtype=torch.uint8, device="cuda")
    base = torch.randn(R, N if epi != 3 else N // 2, device="cuda", generator=g)
    outs = []
    for _ in range(2):
        o = base.clone() if epi in (1, 2) else torch.zeros(R, N // 2 if epi == 3 else N, dtype=torch.bfloat16,
                                                           device="cuda")
        _lib.check(_lib.load().psk_gemv_tc(x.data_ptr(), R, K, hp, mrs.data_ptr(), len(rows), max(rows), N, epi,
                                           o.data_ptr(), ws.data_ptr(), torch.cuda.current_stream().cuda_stream))
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
