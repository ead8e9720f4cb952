"""The reference's TinyLM on the GPU (psk_tiny_forward, fp32, paged prompt
cache) vs the oracle's literal restatement (oracle/tinylm.py, model.ts
:246-412, evaluate.ts:16-50) on identical parameters (same seeded init).
Tolerance: |logit - ref| <= 1e-4 * max|ref| + 1e-5 (fp32 both sides,
different summation order); K/V the same; greedy tokens and sharing
predictions identical."""

import pytest
import torch

import oracle.tinylm as O
from paper_2602_12029_b200 import tinylm as G

pytestmark = pytest.mark.gpu

SMALL = (2, 32, 2, 32, 19)


def _pair(shape, seed, pool=None):
    return G.TinyLM.init(G.TinyConfig(*shape), seed, pool=pool, pool_pages=256), O.TinyLM.init(O.TinyConfig(*shape), seed)


def _prompts(seed, b, n, vocab):
    r = O.Rng(seed)
    return [[r.int(vocab) for _ in range(n)] for _ in range(b)]


def _close(got, ref):
    got = got.detach().float().cpu()
    err = (got - ref).abs().max().item()
    assert err <= 1e-4 * ref.abs().max().item() + 1e-5, err


@pytest.mark.parametrize("shape,b,n", [(SMALL, 2, 7), (SMALL, 3, 32), ((4, 128, 4, 256, 64), 2, 256),
                                       ((2, 64, 4, 64, 40), 4, 50)])
def test_forward_matches_oracle(shape, b, n):
    g, o = _pair(shape, 3)
    toks = _prompts(1, b, n, shape[4])
    gl, gc = g.forward(toks)
    ol, oc = o.forward(toks)
    _close(gl, ol)
    for l in range(shape[0]):
        for r in range(b):
            k, v = gc.kv(l, r)
            _close(k, oc.layers[l][0][r])
            _close(v, oc.layers[l][1][r])


def test_cached_prefix_forward_equals_recompute():
    """model.test.ts:79-101 on the GPU, and each part against the oracle."""
    g, o = _pair(SMALL, 4)
    r = O.Rng(9)
    for _ in range(5):
        prompt = [r.int(19) for _ in range(30)]
        split = 3 + r.int(24)
        full, _ = g.forward([prompt])
        _, pc = g.forward([prompt[:split]])
        rest, rc = g.forward([prompt[split:]], pc)
        assert (full[:, split:] - rest).abs().max().item() < 1e-5
        assert rc.length == 30 and rc.tokens[0] == prompt
        _close(rest, o.forward([prompt[split:]], o.forward([prompt[:split]])[1])[0])


@pytest.mark.parametrize("ratio", [0.0, 0.3, 0.5, 0.77, 1.0])
def test_sharing_predictions_match_oracle(ratio):
    """evaluate.ts:21-50: base cache of the first m positions (sliced
    mid-page), the decode module recomputes the tail over it in place."""
    pool = G.TinyKVPool(G.TinyConfig(*SMALL), 512)
    gb, ob = _pair(SMALL, 1, pool)
    gd, od = _pair(SMALL, 2, pool)
    prompts = _prompts(5, 12, 27, 19)
    assert G.sharing_predictions(gd, gb, ratio, prompts) == O.evaluate_sharing_predictions(od, ob, ratio, prompts)
    targets = O.evaluate_sharing_predictions(od, ob, ratio, prompts)
    assert G.evaluate_sharing(gd, gb, ratio, list(zip(prompts, targets))) == 1.0


def test_copy_on_write_keeps_the_base_cache():
    """Two decode modules append to the same sliced base cache (a partial
    page at the slice point): each gets a private copy of that page, the base
    cache is unchanged, and both match a forward over an unshared cache."""
    pool = G.TinyKVPool(G.TinyConfig(*SMALL), 256)
    gb, _ = _pair(SMALL, 1, pool)
    gd1, od1 = _pair(SMALL, 2, pool)
    gd2, od2 = _pair(SMALL, 3, pool)
    prompts = _prompts(7, 2, 25, 19)
    base = G.build_base_cache(gb, prompts)
    before = [base.kv(l, r) for l in range(2) for r in range(2)]
    past = base.slice(20)  # page 0 whole, page 1 partial (positions 16-19)
    tails = [p[20:] for p in prompts]
    l1, c1 = gd1.forward(tails, past)
    l2, c2 = gd2.forward(tails, past)
    after = [base.kv(l, r) for l in range(2) for r in range(2)]
    for (k0, v0), (k1, v1) in zip(before, after):
        assert torch.equal(k0, k1) and torch.equal(v0, v1)
    for r in range(2):
        assert c1.tables[r][0] == base.tables[r][0] == c2.tables[r][0]  # the whole page is read in place
        assert len({c1.tables[r][1], c2.tables[r][1], base.tables[r][1]}) == 3  # the partial one copied
    ob = O.TinyLM.init(O.TinyConfig(*SMALL), 1)
    opast = O.build_base_cache(ob, prompts).slice(20)
    _close(l1, od1.forward(tails, opast)[0])
    _close(l2, od2.forward(tails, opast)[0])


@pytest.mark.parametrize("incremental", [True, False])
def test_generate_matches_oracle(incremental):
    g, o = _pair(SMALL, 6)
    prompt = _prompts(3, 1, 9, 19)[0]
    assert G.generate(g, prompt, 12, incremental) == O.generate(o, prompt, 12, incremental)


def test_generate_from_injected_base_cache():
    """model.ts:363-412 with a strict-prefix cache from another module's pages."""
    pool = G.TinyKVPool(G.TinyConfig(*SMALL), 256)
    gb, ob = _pair(SMALL, 1, pool)
    gd, od = _pair(SMALL, 2, pool)
    prompt = _prompts(4, 1, 20, 19)[0]
    gp = G.build_base_cache(gb, [prompt]).row(0).slice(13)
    op = O.build_base_cache(ob, [prompt]).row(0).slice(13)
    assert G.generate(gd, prompt, 10, True, gp) == O.generate(od, prompt, 10, True, op)


def test_errors_as_the_reference():
    g, _ = _pair(SMALL, 3)
    with pytest.raises(ValueError):
        g.forward([[1, 2], [3]])
    with pytest.raises(ValueError):
        g.forward([[1] * 33])
    cache = G.build_base_cache(g, [[1, 2, 3]])
    with pytest.raises(ValueError):
        g.forward([[4], [5]], cache)
    with pytest.raises(ValueError):
        G.generate(g, [1, 2, 3], 2, True, cache)
    with pytest.raises(ValueError):
        cache.slice(4)
    with pytest.raises(ValueError):
        G.sharing_predictions(g, g, 0.5, [])


def test_base_cache_slice_property():
    """model.test.ts:125-142 on the GPU: the cache of x equals the cache of
    x + suffix sliced to len(x)."""
    g, _ = _pair(SMALL, 6)
    r = O.Rng(4)
    x, suf = [r.int(19) for _ in range(20)], [r.int(19) for _ in range(5)]
    short, long = G.build_base_cache(g, [x]), G.build_base_cache(g, [x + suf]).slice(20)
    assert long.tokens[0] == x
    for l in range(SMALL[0]):
        (ks, vs), (kl, vl) = short.kv(l), long.kv(l)
        assert (ks - kl).abs().max().item() < 1e-5 and (vs - vl).abs().max().item() < 1e-5


def test_incremental_equals_full_and_injected_prefix():
    """model.test.ts:167-191 and A9 (acceptance.test.ts:75-92, reduced) on the GPU."""
    g, _ = _pair(SMALL, 8)
    r = O.Rng(7)
    for _ in range(6):
        prompt = [r.int(19) for _ in range(4 + r.int(20))]
        assert G.generate(g, prompt, 6, incremental=True) == G.generate(g, prompt, 6, incremental=False)
    prompt = [r.int(19) for _ in range(22)]
    cache = G.build_base_cache(g, [prompt])
    assert G.generate(g, prompt, 5, past=cache.slice(6)) == G.generate(g, prompt, 5)
    assert G.generate(g, prompt, 5, past=cache.slice(17)) == G.generate(g, prompt, 5)
    assert G.generate(g, [1, 2, 3], 0) == []


def test_evaluate_sharing_contract():
    """evaluate.test.ts:9-47 on the GPU: r = 0 is the decode model alone;
    r = 1 with dec = base equals the base alone."""
    pool = G.TinyKVPool(G.TinyConfig(*SMALL), 512)
    base, dec = _pair(SMALL, 0, pool)[0], _pair(SMALL, 1, pool)[0]
    r = O.Rng(42)
    prompts = [[r.int(19) for _ in range(9)] for _ in range(8)]
    own = [G.generate(dec, p, 1)[0] for p in prompts]
    assert G.sharing_predictions(dec, base, 0, prompts) == own
    assert G.sharing_predictions(base, base, 1, prompts) == G.sharing_predictions(base, base, 0, prompts)


def test_cache_from_another_pool():
    """Models built without a shared pool still consume each other's caches
    (model.ts caches are plain tensors): the pages are imported."""
    gb, ob = _pair(SMALL, 1)
    gd, od = _pair(SMALL, 2)
    assert gb.pool is not gd.pool
    prompts = _prompts(5, 4, 27, 19)
    for ratio in (0.3, 0.77):
        assert G.sharing_predictions(gd, gb, ratio, prompts) == O.evaluate_sharing_predictions(od, ob, ratio, prompts)


@pytest.mark.parametrize("shape,n", [((2, 128, 1, 256, 30), 256), ((1, 64, 2, 40, 11), 40)])
def test_wide_heads_and_full_context(shape, n):
    """One 128-dim head at a 256-token context (K / V read from the pages:
    too large to stage in shared memory) and a forward filling the context
    exactly, then one more token over the cache at the limit - 1."""
    g, o = _pair(shape, 9)
    toks = _prompts(2, 2, n, shape[4])
    gl, gc = g.forward(toks)
    ol, oc = o.forward(toks)
    _close(gl, ol)
    gl2, _ = g.forward([[1], [2]], gc.slice(n - 1))
    _close(gl2, o.forward([[1], [2]], oc.slice(n - 1))[0])
