"""tcgen05 GEMM (K1) and its fused epilogues (K2) vs a torch fp32 reference
on the same bf16 operands. Tolerance: fp32 accumulation of bf16 products;
outputs rounded to bf16 where the kernel stores bf16:
  |gpu - ref| <= 1e-2 * max|ref| + 1e-3  (bf16 outputs)
  |gpu - ref| <= 2e-3 * max|ref| + 1e-4  (fp32 outputs)"""

import ctypes as C
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2602_12029_b200 import _lib
    return _lib


def _rand(*shape, std=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * std).to(torch.bfloat16)


@pytest.fixture
def split_ws():
    """Bind the split-K workspace for the test, unbind afterwards."""
    L = _lib()
    L.bind_gemm_workspace(torch.device("cuda", 0))
    yield
    L.check(L.load().psk_gemm_bind_workspace(None, 0))
    L._gemm_ws = None


def _gemm(A, B, epi, out, ldo):
    L = _lib()
    L.check(L.load().psk_gemm(A.data_ptr(), B.data_ptr(), A.shape[0], B.shape[0], A.shape[1], epi,
                              out.data_ptr(), ldo, torch.cuda.current_stream().cuda_stream))


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1, 256, 256), (300, 512, 256),
                                   (4096, 6144, 4096), (1000, 1024, 14336), (129, 4096, 4096),
                                   (9000, 1024, 512), (12288, 2048, 256)])
def test_gemm_store(M, N, K):
    A, B = _rand(M, K, seed=1), _rand(N, K, std=0.02, seed=2)
    ref = A.float() @ B.float().T
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    _gemm(A, B, 1, out, N)
    torch.cuda.synchronize()
    scale = ref.abs().max().item()
    assert (out - ref).abs().max().item() <= 2e-3 * scale + 1e-4
    outb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, 0, outb, N)
    torch.cuda.synchronize()
    assert (outb.float() - ref).abs().max().item() <= 1e-2 * scale + 1e-3


def test_gemm_residual_add():
    M, N, K = 513, 512, 1024
    A, B = _rand(M, K, seed=3), _rand(N, K, std=0.02, seed=4)
    h = torch.randn(M, N, device="cuda")
    ref = h + A.float() @ B.float().T
    _gemm(A, B, 2, h, N)
    torch.cuda.synchronize()
    assert (h - ref).abs().max().item() <= 2e-3 * ref.abs().max().item() + 1e-4


def test_gemm_silu_mul_interleaved():
    M, F, K = 200, 768, 256
    A = _rand(M, K, seed=5)
    Wg, Wu = _rand(F, K, std=0.05, seed=6), _rand(F, K, std=0.05, seed=7)
    Wgu = torch.stack([Wg.view(-1, 8, K), Wu.view(-1, 8, K)], 1).reshape(2 * F, K).contiguous()
    ref = torch.nn.functional.silu(A.float() @ Wg.float().T) * (A.float() @ Wu.float().T)
    out = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    _gemm(A, Wgu, 3, out, F)
    torch.cuda.synchronize()
    assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("nq,nkv,T,pos0", [(2, 1, 100, 0), (32, 8, 300, 32), (32, 8, 17, 4080), (32, 8, 4096, 16)])
def test_gemm_qkv_rope_paged_kv(nq, nkv, T, pos0):
    """(T = 4096 at the 8B width: 768 tiles, the last-wave tiles run as
    128-column (one head) pieces: split-N.)"""
    _qkv_case(nq, nkv, T, pos0)


def test_gemm_qkv_rope_paged_kv_split_k(split_ws):
    """The same with the split-K workspace bound."""
    _qkv_case(32, 8, 4096, 16)


def _qkv_case(nq, nkv, T, pos0):
    from paper_2602_12029_b200.model import KVCache, LlamaConfig, rope_table
    from oracle.model import _rope, rope_cos_sin
    d = 256 if nq == 2 else 4096
    cfg = LlamaConfig(n_layers=2, d_model=d, n_heads=nq, n_kv_heads=nkv, ffn=768, vocab=512,
                      rope_theta=5e5, max_pos=8192)
    A = _rand(T, d, seed=8)
    W = _rand(cfg.qkv_dim, d, std=0.02, seed=9)
    n_pages = (pos0 + T + 15) // 16
    pages = list(np.random.default_rng(0).permutation(n_pages + 5)[:n_pages])
    kv = KVCache(cfg, n_pages + 5)
    rope = torch.from_numpy(rope_table(cfg)).cuda()
    pt = torch.tensor(pages, dtype=torch.int32, device="cuda")
    q = torch.empty(T, nq, 128, dtype=torch.bfloat16, device="cuda")
    L = _lib()
    L.check(L.load().psk_gemm_qkv_rope_kv(A.data_ptr(), W.data_ptr(), T, d, nq, rope.data_ptr(), pos0,
                                          kv.layout(), 1, pt.data_ptr(), q.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    qkv = (A.float() @ W.float().T).cpu()
    cos, sin = rope_cos_sin(8192, 128, 5e5)
    cs, sn = cos[pos0:pos0 + T], sin[pos0:pos0 + T]
    rq = _rope(qkv[:, :nq * 128].view(T, nq, 128).transpose(0, 1), cs, sn)
    rk = _rope(qkv[:, nq * 128:(nq + nkv) * 128].view(T, nkv, 128).transpose(0, 1), cs, sn)
    rv = qkv[:, (nq + nkv) * 128:].view(T, nkv, 128).transpose(0, 1)
    gq = q.float().cpu().transpose(0, 1)
    gk, gv = kv.read_positions(pages, 1, T, start=pos0)
    for got, want in ((gq, rq), (gk.float().cpu(), rk), (gv.float().cpu(), rv)):
        assert (got - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-3
    # layer 0 untouched
    k0, _ = kv.read_positions(pages, 0, T, start=pos0)
    assert k0.abs().max().item() == 0


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 4096), (4096, 6144, 4096), (2560, 2048, 4096),
                                   (4096, 4096, 14336), (4000, 4096, 1024)])
def test_gemm_split_k_tail(M, N, K, split_ws):
    """Last-wave tiles split along K (workspace bound): store / residual add /
    SiLU*mul epilogues; repeated launches (the tail counters re-arm)."""
    A, B = _rand(M, K, seed=11), _rand(N, K, std=0.02, seed=12)
    ref = A.float() @ B.float().T
    scale = ref.abs().max().item()
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    for _ in range(2):
        _gemm(A, B, 1, out, N)
    torch.cuda.synchronize()
    assert (out - ref).abs().max().item() <= 2e-3 * scale + 1e-4
    h = torch.randn(M, N, device="cuda")
    want = h + ref
    _gemm(A, B, 2, h, N)
    torch.cuda.synchronize()
    assert (h - want).abs().max().item() <= 2e-3 * want.abs().max().item() + 1e-4
    F = N // 2
    silu_ref = ref.view(M, -1, 2, 8)
    silu_ref = (torch.nn.functional.silu(silu_ref[:, :, 0]) * silu_ref[:, :, 1]).reshape(M, F)
    o = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, 3, o, F)
    torch.cuda.synchronize()
    assert (o.float() - silu_ref).abs().max().item() <= 1e-2 * silu_ref.abs().max().item() + 1e-3
    assert int(_lib()._gemm_ws[:4096].view(torch.int32).abs().sum().item()) == 0


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 4096), (4096, 6144, 4096), (2560, 2048, 4096),
                                   (4096, 28672, 4096), (4000, 4096, 1024)])
def test_gemm_split_n_tail(M, N, K):
    """Default tail schedule (no workspace): last-wave tiles split along N
    into 64/128-column pieces; store / residual add / SiLU*mul epilogues."""
    assert _lib()._gemm_ws is None
    A, B = _rand(M, K, seed=21), _rand(N, K, std=0.02, seed=22)
    ref = A.float() @ B.float().T
    scale = ref.abs().max().item()
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    _gemm(A, B, 1, out, N)
    torch.cuda.synchronize()
    assert (out - ref).abs().max().item() <= 2e-3 * scale + 1e-4
    h = torch.randn(M, N, device="cuda")
    want = h + ref
    _gemm(A, B, 2, h, N)
    torch.cuda.synchronize()
    assert (h - want).abs().max().item() <= 2e-3 * want.abs().max().item() + 1e-4
    F = N // 2
    silu_ref = ref.view(M, -1, 2, 8)
    silu_ref = (torch.nn.functional.silu(silu_ref[:, :, 0]) * silu_ref[:, :, 1]).reshape(M, F)
    o = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    _gemm(A, B, 3, o, F)
    torch.cuda.synchronize()
    assert (o.float() - silu_ref).abs().max().item() <= 1e-2 * silu_ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("M,N,K", [(300, 512, 256), (257, 6144, 4096), (4096, 6144, 4096), (2560, 2048, 4096)])
def test_gemm_pair_matches_one_sm(M, N, K, tmp_path):
    """The CTA-pair kernel (default) and the 1-SM kernel (PSK_GEMM_PAIR=0,
    read once per process, so it runs in a child) are the same fp32 sums in
    the same k order per output: bit-identical fp32 outputs, fully
    out-of-range second-CTA rows included (M=257, 300)."""
    import os
    import subprocess
    import sys
    A, B = _rand(M, K, seed=31), _rand(N, K, std=0.02, seed=32)
    out = torch.empty(M, N, dtype=torch.float32, device="cuda")
    _gemm(A, B, 1, out, N)
    torch.cuda.synchronize()
    torch.save({"A": A.cpu(), "B": B.cpu()}, tmp_path / "ab.pt")
    code = ("import sys, torch; sys.path.insert(0, %r); from paper_2602_12029_b200 import _lib; L = _lib.load();"
            "d = torch.load(%r); A, B = d['A'].cuda(), d['B'].cuda();"
            "o = torch.empty(A.shape[0], B.shape[0], dtype=torch.float32, device='cuda');"
            "_lib.check(L.psk_gemm(A.data_ptr(), B.data_ptr(), A.shape[0], B.shape[0], A.shape[1], 1, o.data_ptr(),"
            " B.shape[0], torch.cuda.current_stream().cuda_stream)); torch.save(o.cpu(), %r)"
            % (str(Path(__file__).resolve().parent.parent), str(tmp_path / "ab.pt"), str(tmp_path / "o.pt")))
    env = dict(os.environ, PSK_GEMM_PAIR="0")
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=300)
    one_sm = torch.load(tmp_path / "o.pt")
    assert torch.equal(out.cpu(), one_sm)
