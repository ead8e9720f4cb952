"""The literal TinyLM/Rng restatement (oracle/tinylm.py) against the
reference's own golden vectors (rng.test.ts:5-13) and property tests
(model.test.ts:16-191, evaluate.test.ts:9-47, acceptance A9)."""

import pytest
import torch

from oracle.tinylm import (Rng, TinyConfig, TinyLM, build_base_cache, evaluate_sharing_predictions,
                           generate, mix_seed, shared_prefix_length, splitmix64)

CFG = TinyConfig(layers=2, width=32, heads=2, context=32, vocab=19)


def _prompt(rng, n, vocab=CFG.vocab):
    return [rng.int(vocab) for _ in range(n)]


def test_splitmix64_published_vectors():
    s, out = 0, []
    for _ in range(3):
        s, z = splitmix64(s)
        out.append(z)
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_rng_and_mix_seed_properties():
    a, b = Rng(42), Rng(42)
    assert [a.float() for _ in range(50)] == [b.float() for _ in range(50)]
    r = Rng(3)
    assert all(0 <= r.int(7) < 7 for _ in range(500))
    with pytest.raises(ValueError):
        r.int(0)
    assert mix_seed(1, "a", "b") != mix_seed(1, "b", "a")
    assert mix_seed(1, "ab") != mix_seed(1, "a", "b")
    assert mix_seed(9, "train") == mix_seed(9, "train")
    g = Rng(11)
    xs = [g.gauss() for _ in range(20000)]
    m = sum(xs) / len(xs)
    assert abs(m) < 0.03 and abs(sum(x * x for x in xs) / len(xs) - m * m - 1) < 0.05


def test_init_deterministic_and_width_check():
    a, b, c = TinyLM.init(CFG, 5), TinyLM.init(CFG, 5), TinyLM.init(CFG, 6)
    assert torch.equal(a.p["head"], b.p["head"]) and not torch.equal(a.p["head"], c.p["head"])
    with pytest.raises(ValueError):
        TinyLM.init(TinyConfig(2, 30, 4, 32, 19), 0)


def test_forward_shapes_and_errors():
    m = TinyLM.init(CFG, 3)
    logits, cache = m.forward([_prompt(Rng(0), 7), _prompt(Rng(1), 7)])
    assert logits.shape == (2, 7, CFG.vocab) and cache.length == 7 and cache.batch == 2
    with pytest.raises(ValueError):
        m.forward([[1, 2], [3]])
    with pytest.raises(ValueError):
        m.forward([_prompt(Rng(0), CFG.context + 1)])
    cache = build_base_cache(m, [[1, 2, 3]])
    with pytest.raises(ValueError):
        m.forward([[4], [5]], cache)


def test_cached_prefix_forward_equals_recompute():
    """model.test.ts:79-101."""
    m = TinyLM.init(CFG, 4)
    rng = Rng(9)
    for _ in range(5):
        prompt = _prompt(rng, 12)
        split = 3 + rng.int(8)
        full, fc = m.forward([prompt])
        _, pc = m.forward([prompt[:split]])
        rest, rc = m.forward([prompt[split:]], pc)
        assert (full[:, split:] - rest).abs().max() < 1e-5
        assert rc.length == 12 and rc.tokens[0] == prompt
        for l in range(CFG.layers):
            assert (fc.layers[l][0] - rc.layers[l][0]).abs().max() < 1e-5
            assert (fc.layers[l][1] - rc.layers[l][1]).abs().max() < 1e-5


def test_base_cache_slice_property():
    """model.test.ts:125-142."""
    m = TinyLM.init(CFG, 6)
    rng = Rng(4)
    x, suf = _prompt(rng, 8), _prompt(rng, 5)
    short, long = build_base_cache(m, [x]), build_base_cache(m, [x + suf]).slice(8)
    assert long.tokens[0] == x
    for l in range(CFG.layers):
        assert (short.layers[l][0] - long.layers[l][0]).abs().max() < 1e-5
        assert (short.layers[l][1] - long.layers[l][1]).abs().max() < 1e-5


def test_prompt_cache_slice_row_validation():
    """model.test.ts:146-164."""
    m = TinyLM.init(CFG, 7)
    prompts = [_prompt(Rng(5), 6), _prompt(Rng(6), 6)]
    cache = build_base_cache(m, prompts)
    for bad in (lambda: cache.slice(7), lambda: cache.slice(-1), lambda: cache.row(2)):
        with pytest.raises(ValueError):
            bad()
    assert cache.row(1).tokens[0] == prompts[1] and cache.slice(4).tokens == [p[:4] for p in prompts]


def test_incremental_equals_full_and_injected_prefix():
    """model.test.ts:167-191 and A9 (acceptance.test.ts:75-92, reduced)."""
    m = TinyLM.init(CFG, 8)
    rng = Rng(7)
    for _ in range(6):
        prompt = _prompt(rng, 4 + rng.int(8))
        assert generate(m, prompt, 6, incremental=True) == generate(m, prompt, 6, incremental=False)
    prompt = _prompt(Rng(8), 10)
    cache = build_base_cache(m, [prompt])
    assert generate(m, prompt, 5, past=cache.slice(6)) == generate(m, prompt, 5)
    with pytest.raises(ValueError):
        generate(m, prompt, 3, past=cache)
    assert generate(m, [1, 2, 3], 0) == []


def test_evaluate_sharing_contract():
    """evaluate.ts:16-50 / evaluate.test.ts:9-47: the decode model processes
    the last prompt token itself; r=0 is the model alone; r=1 with dec=base
    equals the base alone."""
    assert [shared_prefix_length(r, 10) for r in (0, 0.25, 0.5, 1, 0.99)] == [0, 3, 5, 9, 9]
    for bad in (-0.1, 1.1, float("nan")):
        with pytest.raises(ValueError):
            shared_prefix_length(bad, 10)
    base, dec = TinyLM.init(CFG, 0), TinyLM.init(CFG, 1)
    rng = Rng(42)
    prompts = [_prompt(rng, 9) for _ in range(8)]
    own = [generate(dec, p, 1)[0] for p in prompts]
    assert evaluate_sharing_predictions(dec, base, 0, prompts) == own
    assert evaluate_sharing_predictions(base, base, 1, prompts) == evaluate_sharing_predictions(base, base, 0, prompts)
