"""K5-TC QKV projection with RoPE + KV append fused into its epilogue
(psk_gemv_tc_qkv_rope) vs the two-kernel path it replaces
(psk_gemv_tc(PSK_EPI_STORE_F32) + psk_rope_append) on identical inputs:
q_rot and every KV page bit-identical, and the whole decode step (CUDA
graph, DecodeRunner) producing bit-identical logits and tokens with the
fusion on and off. Rows per module 9..64 (all three K5-TC tile widths),
ragged, modules without rows, private lengths crossing page boundaries."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _batch(cfg, rows_per_mod, seed):
    from paper_2602_12029_b200.model import DecodeBatch, DecodeRow, KVCache, SessionSpec
    rng = np.random.default_rng(seed)
    n_mod = len(rows_per_mod)
    R = sum(rows_per_mod)
    # one session per row (agent-serving layout), shared prefixes of random length
    sess_lens = [int(x) for x in rng.integers(0, 300, R)]
    priv = [int(x) for x in rng.integers(0, 40, R)]
    n_pages = sum((L + 15) // 16 for L in sess_lens) + sum(p // 16 + 1 for p in priv) + 4
    kv = KVCache(cfg, n_pages)
    perm = list(rng.permutation(n_pages))
    sessions, rows = [], []
    ri = 0
    for m, nr in enumerate(rows_per_mod):
        for _ in range(nr):
            L = sess_lens[ri]
            sessions.append(SessionSpec(shared_len=L, pages=[perm.pop() for _ in range(max(1, (L + 15) // 16))]))
            rows.append(DecodeRow(module=m, session=ri, first_token=0,
                                  pages=[perm.pop() for _ in range(priv[ri] // 16 + 1)]))
            ri += 1
    b = DecodeBatch(sessions, rows, n_mod)
    b.t_priv_len.copy_(torch.tensor([priv[j] for j in b.order], dtype=torch.int32))
    return b, kv


@pytest.mark.parametrize("rows_per_mod", [[9, 12, 0, 10], [20, 32, 17], [40, 64], [33]])
def test_fused_qkv_rope_bit_identical(rows_per_mod):
    from paper_2602_12029_b200 import _lib
    from paper_2602_12029_b200.model import LlamaConfig, rope_table
    cfg = LlamaConfig(n_layers=3, d_model=512, n_heads=8, n_kv_heads=2, ffn=256, vocab=64, rope_theta=1e4,
                      max_pos=1024)
    b, kv = _batch(cfg, rows_per_mod, seed=sum(rows_per_mod))
    g = torch.Generator(device="cuda").manual_seed(len(rows_per_mod))
    n_mod, R, d, N = len(rows_per_mod), b.n_rows, cfg.d_model, cfg.qkv_dim
    W = [(torch.randn(N, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16) for _ in range(n_mod)]
    hp = (ctypes.c_void_p * n_mod)(*[w.data_ptr() for w in W])
    x = torch.randn(R, d, device="cuda", generator=g).to(torch.bfloat16)
    rope = torch.from_numpy(rope_table(cfg)).cuda()
    lib = _lib.load()
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_gemv_tc_workspace(ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    layer = 1
    kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
    kv0 = kv.data.clone()
    # two-kernel path
    qkv = torch.empty(R, N, device="cuda")
    q_a = torch.full((R, cfg.n_heads, 128), float("nan"), device="cuda").to(torch.bfloat16)
    _lib.check(lib.psk_gemv_tc(x.data_ptr(), R, d, hp, b.t_mrs.data_ptr(), n_mod, b.max_rpm, N, 1,
                               qkv.data_ptr(), ws.data_ptr(), s))
    _lib.check(lib.psk_rope_append(b.c_ref(), qkv.data_ptr(), cfg.n_heads, rope.data_ptr(), layer, kv.layout(),
                                   q_a.data_ptr(), s))
    torch.cuda.synchronize()
    kv_a = kv.data.clone()
    # fused
    kv.data.copy_(kv0)
    q_b = torch.full_like(q_a, float("nan"))
    for _ in range(2):  # twice: the stream-K flags come back zeroed
        _lib.check(lib.psk_gemv_tc_qkv_rope(x.data_ptr(), d, hp, b.c_ref(), b.max_rpm, cfg.n_heads, rope.data_ptr(),
                                            layer, kv.layout(), q_b.data_ptr(), ws.data_ptr(), s))
    torch.cuda.synchronize()
    assert int(ws[:4096].view(torch.int32).abs().sum().item()) == 0
    assert torch.equal(q_a.view(torch.int16), q_b.view(torch.int16))
    assert torch.equal(kv_a.view(torch.int16), kv.data.view(torch.int16))
    assert not torch.equal(kv_a, kv0)  # the append happened


@pytest.mark.parametrize("rows", [12, 40])
def test_decode_step_fused_qkv_same_tokens(rows, monkeypatch):
    """DecodeRunner (graph-replayed steps) with PSK_FUSED_QKV on / off:
    logits and generated tokens bit-identical."""
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, DecodeRunner, KVCache, LlamaConfig,
                                             ModuleWeights, SessionSpec)
    cfg = LlamaConfig.tiny()
    mods = [ModuleWeights(cfg, 11 + i) for i in range(2)]
    out = []
    S = rows  # sessions, each decoded by both modules: `rows` rows per module
    for fused in ("1", "0"):
        monkeypatch.setenv("PSK_FUSED_QKV", fused)
        kv = KVCache(cfg, 4 * S + 2 * S)
        g = torch.Generator(device="cuda").manual_seed(3)
        kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
        sess = [SessionSpec(shared_len=40 + s % 24, pages=list(range(4 * s, 4 * s + 4))) for s in range(S)]
        rws = [DecodeRow(module=m, session=s, first_token=5 + s + m, pages=[4 * S + 2 * s + m])
               for s in range(S) for m in range(2)]
        b = DecodeBatch(sess, rws, 2)
        r = DecodeRunner(cfg, mods, kv, b, 8)
        assert r.use_tc_gemv and r.fused_qkv == (fused == "1")
        toks = r.run(8)
        torch.cuda.synchronize()
        out.append((toks.clone(), r.logits.clone(), kv.data.clone()))
    assert torch.equal(out[0][0], out[1][0])  # (fused, unfused)
    assert torch.equal(out[0][1], out[1][1])
    assert torch.equal(out[0][2].view(torch.int16), out[1][2].view(torch.int16))


@pytest.mark.parametrize("rows", [12, 40])
def test_decode_step_fused_norm_close(rows, monkeypatch):
    """PSK_FUSED_NORM=1 (residual GEMV + next RMSNorm in one launch, grid
    barrier over a module's units) vs the separate norm kernels: the sums of
    squares add in another order, so logits agree to bf16 rounding, and the
    greedy tokens agree except at near-ties."""
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, DecodeRunner, KVCache, LlamaConfig,
                                             ModuleWeights, SessionSpec)
    cfg = LlamaConfig.tiny()
    mods = [ModuleWeights(cfg, 11 + i) for i in range(2)]
    out = []
    S = rows
    for fused in ("1", "0"):
        monkeypatch.setenv("PSK_FUSED_NORM", fused)
        kv = KVCache(cfg, 4 * S + 2 * S)
        g = torch.Generator(device="cuda").manual_seed(3)
        kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
        sess = [SessionSpec(shared_len=40 + s % 24, pages=list(range(4 * s, 4 * s + 4))) for s in range(S)]
        rws = [DecodeRow(module=m, session=s, first_token=5 + s + m, pages=[4 * S + 2 * s + m])
               for s in range(S) for m in range(2)]
        r = DecodeRunner(cfg, mods, kv, DecodeBatch(sess, rws, 2), 8)
        assert r.fused_norm == (fused == "1")
        r.run(1)
        torch.cuda.synchronize()
        out.append(r.logits.clone())
    a, b = out
    assert (a - b).abs().max().item() <= 2e-2 * b.abs().max().item()
