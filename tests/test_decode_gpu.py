"""GPU parity of the decode-module step (K5 GEMV, K6 shared-prefix decode
attention, RoPE/KV append, argmax) against the fp32 Llama oracle.

The base module's prompt KV is produced by the oracle (rounded to bf16, the
storage type of the paged cache) and written into shared pages; every
decode module then generates from it through the GPU path. Tolerances (bf16
weights/activations, fp32 accumulation):
  * first-step logits: max|gpu - oracle| <= 2e-2 * max|oracle logits| + 1e-3
  * greedy tokens: identical under teacher forcing wherever the oracle's
    top-1/top-2 logit margin exceeds 2e-2 * max|logit| (random-init logits are
    nearly flat, so near-ties may legitimately flip).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 2e-2


def _setup(cfg, n_modules, seeds=None):
    from paper_2602_12029_b200.model import ModuleWeights
    from oracle.model import LlamaOracle
    seeds = seeds or list(range(1, n_modules + 2))
    base = ModuleWeights(cfg, seeds[0], with_head=False)
    mods = [ModuleWeights(cfg, s) for s in seeds[1:n_modules + 1]]
    torch.cuda.synchronize()
    base_o = LlamaOracle(cfg, base.reference_layout())
    mods_o = [LlamaOracle(cfg, m.reference_layout()) for m in mods]
    return base, mods, base_o, mods_o


def _bf16(kv):
    return [(k.to(torch.bfloat16).float(), v.to(torch.bfloat16).float()) for k, v in kv]


def _run_case(cfg, prompts, attach, max_new, check_tokens=True):
    """prompts: list of token lists (one per session); attach: list of
    (module, session) decode rows."""
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, DecodeRunner, KVCache,
                                             SessionSpec, PAGE_TOKENS)
    n_mod = max(m for m, _ in attach) + 1
    base, mods, base_o, mods_o = _setup(cfg, n_mod)
    next_page = [0]

    def alloc(n):
        out = list(range(next_page[0], next_page[0] + n))
        next_page[0] += n
        return out

    shared = []
    sess_specs = []
    for p in prompts:
        L = len(p) - 1
        kv = _bf16(base_o.prefill(p[:-1]))
        pages = alloc((L + PAGE_TOKENS - 1) // PAGE_TOKENS)
        shared.append(kv)
        sess_specs.append(SessionSpec(shared_len=L, pages=pages))
    priv_pages = (max_new + PAGE_TOKENS - 1) // PAGE_TOKENS
    rows = [DecodeRow(module=m, session=s, first_token=prompts[s][-1], pages=alloc(priv_pages))
            for m, s in attach]
    kv = KVCache(cfg, next_page[0] + 1)
    for spec, skv in zip(sess_specs, shared):
        for l in range(cfg.n_layers):
            kv.write_positions(spec.pages, l, skv[l][0].cuda(), skv[l][1].cuda())
    batch = DecodeBatch(sess_specs, rows, n_mod)
    runner = DecodeRunner(cfg, mods, kv, batch, max_new)
    # -- first step, eager: logits
    runner.run(1, use_graph=False)
    torch.cuda.synchronize()
    logits = runner.logits.cpu()
    inv = {j: i for i, j in enumerate(batch.order)}  # caller row -> batch row
    want_first = []
    for i, (m, s) in enumerate(attach):
        lg, _ = mods_o[m].forward([prompts[s][-1]], shared[s])
        want_first.append(lg[-1])
        got = logits[inv[i]]
        scale = float(lg[-1].abs().max())
        err = float((got - lg[-1]).abs().max())
        assert err <= LOGIT_RTOL * scale + 1e-3, f"row {i}: logits err {err} (scale {scale})"
    # -- full greedy generation through the CUDA graph
    toks = runner.run(max_new, use_graph=True).cpu().numpy()
    # KV appended by the GPU for the private suffix of row 0, layer 0
    results = []
    for i, (m, s) in enumerate(attach):
        got = toks[i].tolist()
        want, lgs = mods_o[m].generate(prompts[s], max_new, past=shared[s], teacher=got[:-1])
        flips = 0
        for t in range(max_new):
            lg = lgs[t]
            top2 = torch.topk(lg, 2).values
            margin = float(top2[0] - top2[1])
            if got[t] != want[t]:
                flips += 1
                assert margin <= LOGIT_RTOL * float(lg.abs().max()), \
                    f"row {i} step {t}: token {got[t]} != {want[t]} with margin {margin}"
        results.append((got, want, flips))
    return runner, results


def test_tiny_single_session_two_modules():
    """BASELINE config 1 shape: tiny Llama, 2 decode modules on one shared prompt."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.tiny()
    rng = np.random.default_rng(0)
    prompt = rng.integers(0, cfg.vocab, 100).tolist()
    _, res = _run_case(cfg, [prompt], [(0, 0), (1, 0)], max_new=24)
    assert sum(f for _, _, f in res) <= 2


def test_tiny_multi_session_multi_row_modules():
    """2 sessions x 2 modules (2 rows per module -> grouped GEMV with M=2),
    ragged prompt lengths incl. one that ends mid-page."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.tiny()
    rng = np.random.default_rng(1)
    prompts = [rng.integers(0, cfg.vocab, 100).tolist(), rng.integers(0, cfg.vocab, 37).tolist()]
    _, res = _run_case(cfg, prompts, [(0, 0), (1, 0), (0, 1), (1, 1)], max_new=20)
    assert sum(f for _, _, f in res) <= 3


def test_tiny_sixteen_modules_one_session():
    """Config-4 fan-out shape at tiny width: 16 decode modules share one prompt
    (64 query rows per KV head in the shared pass)."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.tiny()
    rng = np.random.default_rng(2)
    prompt = rng.integers(0, cfg.vocab, 300).tolist()
    _, res = _run_case(cfg, [prompt], [(m, 0) for m in range(16)], max_new=6)
    assert sum(f for _, _, f in res) <= 3


def test_8b_shape_two_layer_truncation():
    """Llama-3.1-8B width (d=4096, 32q/8kv, ffn 14336, vocab 128256), 2 layers,
    4 decode modules sharing one prompt."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.llama8b(n_layers=2, max_pos=1024)
    rng = np.random.default_rng(3)
    prompt = rng.integers(0, cfg.vocab, 200).tolist()
    _, res = _run_case(cfg, [prompt], [(m, 0) for m in range(4)], max_new=8)
    assert sum(f for _, _, f in res) <= 2


def test_tiny_twelve_rows_per_module_tc_gemv():
    """12 sessions x 2 modules = 12 rows per module: the decode GEMVs run on
    the tcgen05 kernel (K5-TC, MN = 16)."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.tiny()
    rng = np.random.default_rng(4)
    prompts = [rng.integers(0, cfg.vocab, int(n)).tolist() for n in rng.integers(5, 120, 12)]
    attach = [(m, s) for s in range(12) for m in range(2)]
    runner, res = _run_case(cfg, prompts, attach, max_new=6)
    assert runner.use_tc_gemv
    assert sum(f for _, _, f in res) <= 4


def test_tiny_forty_rows_one_module_tc_gemv():
    """40 sessions on one decode module (K5-TC with MN = 64)."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.tiny()
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, cfg.vocab, int(n)).tolist() for n in rng.integers(3, 50, 40)]
    runner, res = _run_case(cfg, prompts, [(0, s) for s in range(40)], max_new=4)
    assert runner.use_tc_gemv
    assert sum(f for _, _, f in res) <= 4


def test_8b_shape_twenty_rows_per_module():
    """8B width, 2 layers, 10 sessions x 2 modules (K5-TC, MN = 16 / 32 incl.
    the 128256-row LM head)."""
    from paper_2602_12029_b200.model import LlamaConfig
    cfg = LlamaConfig.llama8b(n_layers=2, max_pos=1024)
    rng = np.random.default_rng(6)
    prompts = [rng.integers(0, cfg.vocab, int(n)).tolist() for n in rng.integers(20, 90, 20)]
    runner, res = _run_case(cfg, prompts, [(m, s) for s in range(20) for m in range(2)], max_new=3)
    assert runner.use_tc_gemv
    assert sum(f for _, _, f in res) <= 4


def test_decode_batch_rejects_short_page_tables():
    """A session whose page list cannot hold its shared length would make the
    kernels read page ids past the table: DecodeBatch refuses it."""
    from paper_2602_12029_b200.model import DecodeBatch, DecodeRow, SessionSpec
    with pytest.raises(ValueError):
        DecodeBatch([SessionSpec(shared_len=65, pages=[0, 1, 2, 3])],
                    [DecodeRow(module=0, session=0, first_token=1, pages=[4])], 1)
    DecodeBatch([SessionSpec(shared_len=64, pages=[0, 1, 2, 3])],
                [DecodeRow(module=0, session=0, first_token=1, pages=[4])], 1)
