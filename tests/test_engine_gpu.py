"""PrefillShareEngine.serve (the public API of the bench's e2e leg): grouped
prefills (run_batch, prefill_group sessions per forward, per-sequence K3 for
long prompts) give exactly the tokens of one prefill per session, including
prefix hits inside the same batch and a second serve that hits the pool."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lens", [[70, 33, 120, 16], [1100, 1040, 1030]])
def test_grouped_prefill_serve_matches_single(lens):
    from paper_2602_12029_b200.engine import PrefillShareEngine
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.tiny(max_pos=1400)
    rng = np.random.default_rng(11)
    prompts = [rng.integers(0, cfg.vocab, n, dtype=np.int64) for n in lens]
    prompts[1][:32] = prompts[0][:32]  # two full shared blocks: an in-batch prefix hit
    kw = dict(n_modules=2, max_sessions=len(lens), max_prompt=max(lens), max_new=8, pool_pages=512, seed=3)
    one = PrefillShareEngine(cfg, prefill_group=1, **kw)
    grp = PrefillShareEngine(cfg, prefill_group=2, modules=one.mods, base=one.base, **kw)
    a, b = one.serve(prompts), grp.serve(prompts)
    assert a.matched == b.matched and a.matched[1] == 32
    assert a.prefill_tokens == b.prefill_tokens
    assert np.array_equal(a.tokens, b.tokens)
    again = grp.serve(prompts)  # every full block cached now
    assert all(m == (n // 16) * 16 or m == ((n - 1) // 16) * 16 for m, n in zip(again.matched, lens))
    assert np.array_equal(again.tokens, a.tokens)
    assert grp.launches_per_serve(len(lens), len(lens)) > grp.launches_per_serve(len(lens), 0)
    torch.cuda.synchronize()
