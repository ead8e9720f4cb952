"""GPU parity of the prefill module (K1 tcgen05 GEMMs, K2 fused RoPE + paged
KV write, K3 causal paged attention) against the fp32 Llama oracle, plus
end-to-end shared-prefill -> multi-module decode.

Tolerance: per layer, max|K_gpu - K_ref| and max|V_gpu - V_ref| <= 3e-2 *
max|ref| (bf16 weights, activations and cache; fp32 accumulation; the error
compounds over layers so deeper layers get the same relative bound)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
KV_RTOL = 3e-2


def _build(cfg, n_mod, seed0=1):
    from paper_2602_12029_b200.model import ModuleWeights
    from oracle.model import LlamaOracle
    base = ModuleWeights(cfg, seed0, with_head=False)
    mods = [ModuleWeights(cfg, seed0 + 1 + i) for i in range(n_mod)]
    torch.cuda.synchronize()
    return base, mods, LlamaOracle(cfg, base.reference_layout()), [
        LlamaOracle(cfg, m.reference_layout()) for m in mods]


def _check_kv(kv, pages, cfg, ref_cache, n, start=0):
    for l in range(cfg.n_layers):
        gk, gv = kv.read_positions(pages, l, n, start=start)
        rk, rv = ref_cache[l][0][:, start:start + n], ref_cache[l][1][:, start:start + n]
        for got, want in ((gk.float().cpu(), rk), (gv.float().cpu(), rv)):
            err = (got - want).abs().max().item()
            assert err <= KV_RTOL * want.abs().max().item(), f"layer {l}: kv err {err}"


@pytest.mark.parametrize("shape,n", [("tiny", 512), ("tiny", 77), ("8b2", 300)])
def test_prefill_kv_matches_oracle(shape, n):
    from paper_2602_12029_b200.model import KVCache, LlamaConfig, PrefillRunner
    cfg = LlamaConfig.tiny() if shape == "tiny" else LlamaConfig.llama8b(n_layers=2, max_pos=1024)
    base, _, base_o, _ = _build(cfg, 0)
    prompt = np.random.default_rng(n).integers(0, cfg.vocab, n).tolist()
    n_pages = (n + 15) // 16
    pages = list(np.random.default_rng(1).permutation(n_pages + 3)[:n_pages])
    kv = KVCache(cfg, n_pages + 3)
    pre = PrefillRunner(cfg, base, kv, max_tokens=n)
    pre.run(torch.tensor(prompt, dtype=torch.int64, device="cuda"), 0,
            torch.tensor(pages, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    _check_kv(kv, pages, cfg, base_o.prefill(prompt), n)


def test_partial_prefill_after_prefix_hit():
    """A block-aligned cached prefix [0, 64) + new tokens [64, 150): the
    partial prefill attends to the cached pages (cluster.py:331-332)."""
    from paper_2602_12029_b200.model import KVCache, LlamaConfig, PrefillRunner
    cfg = LlamaConfig.tiny()
    base, _, base_o, _ = _build(cfg, 0)
    prompt = np.random.default_rng(5).integers(0, cfg.vocab, 150).tolist()
    pages = list(range(3, 3 + 10))
    kv = KVCache(cfg, 16)
    pre = PrefillRunner(cfg, base, kv, max_tokens=150)
    pt = torch.tensor(pages, dtype=torch.int32, device="cuda")
    pre.run(torch.tensor(prompt[:64], dtype=torch.int64, device="cuda"), 0, pt)
    pre.run(torch.tensor(prompt[64:], dtype=torch.int64, device="cuda"), 64, pt)
    torch.cuda.synchronize()
    _check_kv(kv, pages, cfg, base_o.prefill(prompt), 150)


@pytest.mark.parametrize("shape", ["tiny", "8b2"])
def test_shared_prefill_then_decode_modules(shape):
    """The PrefillShare pipeline: one base prefill on the GPU writes the
    shared pages; N decode modules generate from them. Tokens must match the
    oracle pipeline (oracle prefill -> oracle decode) under teacher forcing
    except at near-ties (margin <= 2e-2 * max|logit|)."""
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, DecodeRunner, KVCache,
                                             LlamaConfig, PrefillRunner, SessionSpec)
    cfg = LlamaConfig.tiny() if shape == "tiny" else LlamaConfig.llama8b(n_layers=2, max_pos=1024)
    n_mod, n, max_new = (2, 512, 16) if shape == "tiny" else (4, 257, 8)
    base, mods, base_o, mods_o = _build(cfg, n_mod)
    prompt = np.random.default_rng(11).integers(0, cfg.vocab, n).tolist()
    n_pages = (n + 15) // 16
    priv = (max_new + 15) // 16
    kv = KVCache(cfg, n_pages + n_mod * priv)
    pages = list(range(n_pages))
    pre = PrefillRunner(cfg, base, kv, max_tokens=n)
    pre.run(torch.tensor(prompt, dtype=torch.int64, device="cuda"), 0,
            torch.tensor(pages, dtype=torch.int32, device="cuda"))
    rows = [DecodeRow(module=m, session=0, first_token=prompt[-1],
                      pages=list(range(n_pages + m * priv, n_pages + (m + 1) * priv)))
            for m in range(n_mod)]
    batch = DecodeBatch([SessionSpec(shared_len=n - 1, pages=pages)], rows, n_mod)
    runner = DecodeRunner(cfg, mods, kv, batch, max_new)
    toks = runner.run(max_new).cpu().numpy()
    ref_kv = base_o.prefill(prompt[:-1])
    flips = 0
    for m in range(n_mod):
        got = toks[m].tolist()
        want, lgs = mods_o[m].generate(prompt, max_new, past=ref_kv, teacher=got[:-1])
        for t in range(max_new):
            if got[t] != want[t]:
                flips += 1
                top2 = torch.topk(lgs[t], 2).values
                assert float(top2[0] - top2[1]) <= 2e-2 * float(lgs[t].abs().max())
    assert flips <= n_mod


@pytest.mark.parametrize("shape", ["tiny", "8b2", "8b2-long"])
def test_batched_partial_prefill_bit_identical(shape):
    """run_batch (stacked varlen rows: per-row RoPE position + KV slot in the
    QKV epilogue, one K3 CTA per (sequence, q-block)) writes exactly the KV
    and hidden rows that one run() per sequence writes: partial prefills
    after cached prefixes (pos0 > 0, block-aligned and mid-page tails),
    scattered page tables, sequences longer than one q-block."""
    from paper_2602_12029_b200.model import KVCache, LlamaConfig, ModuleWeights, PrefillRunner
    cfg = LlamaConfig.tiny() if shape == "tiny" else LlamaConfig.llama8b(n_layers=2, max_pos=4096)
    base = ModuleWeights(cfg, 5, with_head=False)
    rng = np.random.default_rng(7)
    specs = [(0, 300), (64, 21), (32, 1), (160, 77)]  # (pos0, new tokens)
    if shape == "8b2-long":  # every sequence >= 1024 new tokens: per-sequence K3 launches
        specs = [(0, 1100), (48, 1030), (0, 1024)]
    max_tokens = max(1024, sum(n for _, n in specs))
    n_pages = sum((p + n + 15) // 16 for p, n in specs) + 4
    perm = rng.permutation(n_pages).tolist()
    seqs, pts = [], []
    for p0, n in specs:
        pt = [perm.pop() for _ in range((p0 + n + 15) // 16)]
        pts.append(pt)
        seqs.append((torch.from_numpy(rng.integers(0, cfg.vocab, n)).cuda(), p0, pt))
    prefix = [torch.from_numpy(rng.integers(0, cfg.vocab, p0)).cuda() for p0, _ in specs]
    outs = []
    for batched in (False, True):
        kv = KVCache(cfg, n_pages)
        kv.data.zero_()
        pre = PrefillRunner(cfg, base, kv, max_tokens=max_tokens)
        for (p0, _), pt, pf in zip(specs, pts, prefix):  # cached prefixes, one sequence each
            if p0:
                pre.run(pf, 0, torch.tensor(pt, dtype=torch.int32, device="cuda"))
        hs = []
        if batched:
            pre.run_batch(seqs)
            off = 0
            for _, n in specs:
                hs.append(pre.h[off:off + n].clone())
                off += n
        else:
            for toks, p0, pt in seqs:
                pre.run(toks, p0, torch.tensor(pt, dtype=torch.int32, device="cuda"))
                hs.append(pre.h[:toks.shape[0]].clone())
        torch.cuda.synchronize()
        outs.append((kv.data.clone(), hs))
    (kv_a, h_a), (kv_b, h_b) = outs
    assert torch.equal(kv_a, kv_b)
    for a, b in zip(h_a, h_b):
        assert torch.equal(a, b)


@pytest.mark.parametrize("batched", [False, True])
def test_kv_only_prefill_writes_identical_kv(batched):
    """kv_only stops after the last layer's QKV GEMM: the KV pages of every
    layer are bit-identical to the full forward's."""
    from paper_2602_12029_b200.model import KVCache, LlamaConfig, ModuleWeights, PrefillRunner
    cfg = LlamaConfig.llama8b(n_layers=3, max_pos=2048)
    base = ModuleWeights(cfg, 8, with_head=False)
    rng = np.random.default_rng(3)
    lens = [1100, 1030] if batched else [777]
    seqs, off = [], 0
    for n in lens:
        pages = list(range(off, off + (n + 15) // 16))
        off += len(pages)
        seqs.append((torch.from_numpy(rng.integers(0, cfg.vocab, n)).cuda(), 0, pages))
    outs = []
    for kv_only in (False, True):
        kv = KVCache(cfg, off + 1)
        kv.data.zero_()
        pre = PrefillRunner(cfg, base, kv, max_tokens=sum(lens))
        if batched:
            pre.run_batch(seqs, kv_only=kv_only)
        else:
            t, p0, pg = seqs[0]
            pre.run(t, p0, torch.tensor(pg, dtype=torch.int32, device="cuda"), kv_only=kv_only)
        torch.cuda.synchronize()
        outs.append(kv.data.clone())
    assert torch.equal(outs[0], outs[1]) and outs[0].abs().sum().item() > 0
