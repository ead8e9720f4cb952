"""CPU: the Llama oracle is pinned to transformers' LlamaForCausalLM
(tests/golden/llama_tiny.npz) and satisfies the reference's KV-cache
properties (frontend/tests/model.test.ts:79-191, acceptance A9)."""

import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
import make_llama_golden as G  # noqa: E402

from oracle.model import LlamaOracle  # noqa: E402


def _oracle():
    cfg = SimpleNamespace(**G.CFG)
    w = G.make_weights()
    t = lambda a: torch.from_numpy(a)  # noqa: E731
    tw = {"embed": t(w["embed"]), "final_norm": t(w["final_norm"]), "head": t(w["head"]),
          "layers": [{k: t(v) for k, v in lw.items()} for lw in w["layers"]]}
    return LlamaOracle(cfg, tw)


def test_oracle_matches_transformers_llama():
    g = np.load(Path(G.OUT))
    o = _oracle()
    prompt = g["prompt"].tolist()
    logits, cache = o.forward(prompt)
    np.testing.assert_allclose(logits.numpy(), g["logits"], atol=2e-5, rtol=1e-4)
    for l in range(2):
        np.testing.assert_allclose(cache[l][0].numpy(), g[f"k{l}"], atol=2e-5, rtol=1e-4)
        np.testing.assert_allclose(cache[l][1].numpy(), g[f"v{l}"], atol=2e-5, rtol=1e-4)
    out, _ = o.generate(prompt, len(g["greedy"]))
    assert out == g["greedy"].tolist()


def test_cached_prefix_forward_equals_recompute():
    """model.test.ts:79-101."""
    o = _oracle()
    rng = np.random.default_rng(9)
    for _ in range(4):
        prompt = rng.integers(0, 512, 12).tolist()
        split = int(rng.integers(3, 11))
        full, fcache = o.forward(prompt)
        _, pcache = o.forward(prompt[:split])
        rest, rcache = o.forward(prompt[split:], pcache)
        assert torch.allclose(full[split:], rest, atol=1e-5)
        for l in range(2):
            assert torch.allclose(fcache[l][0], rcache[l][0], atol=1e-5)
            assert torch.allclose(fcache[l][1], rcache[l][1], atol=1e-5)


def test_base_cache_is_prefix_slice():
    """model.test.ts:125-142: cache(X) == first-n slice of cache([X; suffix])."""
    o = _oracle()
    rng = np.random.default_rng(4)
    x, suf = rng.integers(0, 512, 8).tolist(), rng.integers(0, 512, 5).tolist()
    short, long = o.prefill(x), o.prefill(x + suf)
    for l in range(2):
        assert torch.allclose(short[l][0], long[l][0][:, :8], atol=1e-5)
        assert torch.allclose(short[l][1], long[l][1][:, :8], atol=1e-5)


def test_injected_prefix_generate_and_full_cover_rejected():
    """model.test.ts:179-191 and the decode-module contract (:372-374)."""
    o = _oracle()
    prompt = np.random.default_rng(8).integers(0, 512, 10).tolist()
    cache = o.prefill(prompt)
    prefix = [(k[:, :6], v[:, :6]) for k, v in cache]
    with_cache, _ = o.generate(prompt, 5, past=prefix)
    without, _ = o.generate(prompt, 5)
    assert with_cache == without
    with pytest.raises(ValueError):
        o.generate(prompt, 3, past=cache)
    assert o.generate(prompt, 0) == ([], [])


def test_incremental_equals_full_recompute():
    """model.test.ts:167-177 / A9: incremental greedy == full recompute."""
    o = _oracle()
    rng = np.random.default_rng(7)
    for _ in range(3):
        prompt = rng.integers(0, 512, int(rng.integers(4, 12))).tolist()
        inc, _ = o.generate(prompt, 6)
        full = []
        seq = list(prompt)
        for _ in range(6):
            lg, _ = o.forward(seq)
            full.append(int(torch.argmax(lg[-1])))
            seq.append(full[-1])
        assert inc == full


def test_batched_decode_layer_matches_per_row_layer():
    """oracle.decode_layer_batched (the CPU arm's batched decode step) equals
    layer_forward(T=1) row by row."""
    import torch
    from oracle.model import decode_layer_batched, layer_forward, rope_cos_sin
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig(n_layers=1, d_model=256, n_heads=4, n_kv_heads=2, ffn=512, vocab=64, rope_theta=1e4,
                      max_pos=256)
    g = torch.Generator().manual_seed(0)
    r = lambda *s: torch.randn(*s, generator=g) * 0.05  # noqa: E731
    d, hd = cfg.d_model, cfg.head_dim
    lw = {"attn_norm": 1 + r(d), "wq": r(4 * hd, d), "wk": r(2 * hd, d), "wv": r(2 * hd, d), "wo": r(d, 4 * hd),
          "mlp_norm": 1 + r(d), "w_gate": r(512, d), "w_up": r(512, d), "w_down": r(d, 512)}
    cos, sin = rope_cos_sin(cfg.max_pos, hd, cfg.rope_theta)
    R, S = 3, 37
    x = r(R, d) * 20
    kp, vp = r(R, 2, S, hd) * 20, r(R, 2, S, hd) * 20
    xb, (kb, vb) = decode_layer_batched(cfg, lw, x, kp, vp, cos, sin)
    for i in range(R):
        xi, (ki, vi) = layer_forward(cfg, lw, x[i:i + 1], (kp[i], vp[i]), cos, sin)
        assert torch.allclose(xb[i], xi[0], atol=1e-5, rtol=1e-4)
        assert torch.allclose(kb[i, :, 0], ki[:, S], atol=1e-5) and torch.allclose(vb[i, :, 0], vi[:, S], atol=1e-5)
