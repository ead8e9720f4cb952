"""Oracle parity at the BENCHMARKED configuration, through the product path.

BASELINE configs[1]: Llama-3.1-8B shape (32 layers, d 4096, 32 q / 8 kv
heads, ffn 14336, vocab 128256), one frozen prefill module + 4 decode modules,
4096-token prompts, 256 greedy output tokens. The GPU side is exactly what
bench.py times: PrefillShareEngine.serve (GPU block pool, batched kv_only
prefill over run_batch, graph-replayed decode step, K5-TC GEMVs at 32 rows
per module, K6 shared-prefix attention). Two sessions are served; the second
prompt shares its first 2048 tokens with the first, so it is a prefix hit
whose partial prefill attends to the first session's cached pages.

The oracle (oracle/model.py, fp32 on the host) runs its own independent chain
with the weights streamed one layer at a time (ModuleWeights.layer_reference),
so host memory stays near one layer:
  * base prefill of both prompts -> per-layer K/V compared with the GPU's
    paged KV (every position, every layer);
  * each decode module m, session s: the last prompt token plus the GPU's 255
    generated tokens (teacher forcing) over the ORACLE's base KV [0, n-1) ->
    logits at all 256 positions.
Checked (tolerances stated here and in DESIGN.md §5). Error compounds with
depth in bf16 (measured: the bf16 precision model's KV error grows from 0.2%
at layer 0 to ~4% at layer 31), so every bound is relative to that model,
run in the same test on the same weights:
  * KV, every layer: ||gpu - fp32|| <= 1.25 x ||model - fp32|| + 2e-3 (and
    max-abs <= 1.5 x the model's + 5e-3), both sessions;
  * first-step and last-step logits of every (module, session): the same
    form with factor 1.25;
  * all 256 greedy tokens: gpu token == fp32 argmax unless the fp32 top-1 /
    top-2 margin <= 5e-2 max|logit| (a near-tie), and the flip count stays
    within 1.5 x (x2 sessions) the bf16 model's own flips + 16.
With PSK_PARITY_OUT=<path> the per-layer errors, logit errors and flip
counts are written there as JSON (recorded in DESIGN.md §5).
"""

import json
import os
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

# The GPU vs the fp32 chain, bounded by the error the bf16 PRECISION MODEL
# (oracle layer_forward(bf16_storage=True): the same algorithm with every
# tensor the kernels store in bf16 rounded there) shows vs the fp32 chain:
KV_FRO_K = 1.25      # ||K_gpu - K_ref|| / ||K_ref|| <= 1.25 x the model's + 2e-3 (same for V)
KV_MAX_K = 1.5       # worst element / max|ref|      <= 1.5 x the model's + 5e-3
LOGIT_K = 1.25       # logits, Frobenius and max-abs (max: + 1e-2)
TIE_RTOL = 5e-2      # a greedy flip is allowed only at a top-1/top-2 margin <= 5e-2 max|logit|
FLIP_K = 1.5         # flips <= 1.5 x the bf16 model's flip rate (x2 sessions) + 16


def _gpu_kv(kv, pages, layer, n):
    """[n_kv, n, hd] K and V of positions [0, n) from a page table (vectorised)."""
    pv = kv.page_view()
    idx = torch.as_tensor(pages[:(n + 15) // 16], dtype=torch.long, device=kv.data.device)
    blk = pv[idx, layer]  # [P, 2, n_kv, 16, hd]
    kvh = blk.permute(1, 2, 0, 3, 4).reshape(2, blk.shape[2], -1, blk.shape[-1])[:, :, :n]
    return kvh[0].float().cpu(), kvh[1].float().cpu()


def _worst(a, b):
    return (round(max(a[0], b[0]), 5), round(max(a[1], b[1]), 5))


def _rel(got, want):
    """(max-abs error / max|ref|, Frobenius error / ||ref||)."""
    d = got - want
    return (float(d.abs().max()) / max(float(want.abs().max()), 1e-30),
            float(d.norm()) / max(float(want.norm()), 1e-30))


def test_engine_serve_matches_oracle_at_bench_config():
    from oracle.model import final_logits, layer_forward, rope_cos_sin
    from paper_2602_12029_b200.engine import PrefillShareEngine
    from paper_2602_12029_b200.kvstore import SHARED_NS
    from paper_2602_12029_b200.model import LlamaConfig

    torch.set_num_threads(os.cpu_count() or 1)
    t_start = time.time()
    PROMPT, MAX_NEW, N_MOD, SESSIONS = 4096, 256, 4, 32
    cfg = LlamaConfig.llama8b(max_pos=PROMPT + MAX_NEW + 64)
    eng = PrefillShareEngine(cfg, N_MOD, SESSIONS, PROMPT, MAX_NEW,
                             pool_pages=SESSIONS * (PROMPT // 16) + 64, seed=1)
    eng.capture()
    assert eng.runner.use_tc_gemv and eng.batch.max_rpm == SESSIONS  # the bench's K5-TC path
    rng = np.random.default_rng(2024)
    p0 = rng.integers(0, cfg.vocab, PROMPT, dtype=np.int64)
    p1 = np.concatenate([p0[:PROMPT // 2], rng.integers(0, cfg.vocab, PROMPT // 2, dtype=np.int64)])
    prompts = [p0, p1]
    res = eng.serve(prompts)
    torch.cuda.synchronize()
    assert res.matched == [0, PROMPT // 2] and res.prefill_tokens == [PROMPT, PROMPT // 2]
    # logits of the last step (input = generated token 254 -> output token 255)
    inv = {j: i for i, j in enumerate(eng.batch.order)}  # caller row (s*M+m) -> batch row
    last_gpu = eng.runner.logits.cpu().clone()
    # replay step 0 through the same captured graph: first-step logits
    eng.runner.b.reset()
    eng.runner.graph.replay()
    torch.cuda.synchronize()
    first_gpu = eng.runner.logits.cpu().clone()
    first_tok = eng.runner.out_tokens[:, 0].cpu().clone()
    toks = res.tokens  # [S, M, MAX_NEW]
    for s in range(2):
        for m in range(N_MOD):
            assert int(first_tok[inv[s * N_MOD + m]]) == int(toks[s, m, 0])  # replay is deterministic
    # page tables of the two sessions (pool chains; prompts are block-aligned)
    tables = []
    for p in prompts:
        mt, chain = eng.pool.longest_prefix_match(SHARED_NS, p, 10 ** 9)
        assert mt == PROMPT
        tables.append(chain.slots.tolist())
        eng.pool.release(chain)
    assert tables[0][:PROMPT // 32] == tables[1][:PROMPT // 32]  # the shared prefix is one set of pages

    # ---- oracle: base prefill, layer streamed --------------------------------
    cos, sin = rope_cos_sin(cfg.max_pos, cfg.head_dim, cfg.rope_theta)
    emb = eng.base.embed.cpu().float()
    x0 = emb[torch.from_numpy(p0)]
    x0e = x0.clone()  # bf16 precision-model chain of session 0
    x1 = emb[torch.from_numpy(p1[PROMPT // 2:])]
    del emb
    half = PROMPT // 2
    kv = {"gpu": [], "emu": [], "gpu_vs_emu": [], "gpu_s1": []}
    fails = []  # collected, asserted after the report is written
    base_kv = [[], []]  # per session: per layer (K, V) [n_kv, n-1, hd] for the decode modules
    base_kv_emu = []    # session 0, precision-model chain
    with torch.no_grad():
        for l in range(cfg.n_layers):
            lw = eng.base.layer_reference(l)
            x0, (k0, v0) = layer_forward(cfg, lw, x0, None, cos, sin)
            x0e, (k0e, v0e) = layer_forward(cfg, lw, x0e, None, cos, sin, bf16_storage=True)
            x1, (k1, v1) = layer_forward(cfg, lw, x1, (k0[:, :half], v0[:, :half]), cos, sin)
            del lw
            gk, gv = _gpu_kv(eng.kv, tables[0], l, PROMPT)
            e_gpu = _worst(_rel(gk, k0), _rel(gv, v0))
            e_emu = _worst(_rel(k0e, k0), _rel(v0e, v0))
            kv["gpu"].append(e_gpu)
            kv["emu"].append(e_emu)
            kv["gpu_vs_emu"].append(_worst(_rel(gk, k0e), _rel(gv, v0e)))
            gk1, gv1 = _gpu_kv(eng.kv, tables[1], l, PROMPT)  # session 1's own positions [half, n)
            e1 = _worst(_rel(gk1[:, half:], k1[:, half:]), _rel(gv1[:, half:], v1[:, half:]))
            kv["gpu_s1"].append(e1)
            for tag, e in (("session 0", e_gpu), ("session 1", e1)):
                if not (e[1] <= KV_FRO_K * e_emu[1] + 2e-3 and e[0] <= KV_MAX_K * e_emu[0] + 5e-3):
                    fails.append(f"layer {l} {tag}: KV err (max, fro) {e} vs bf16 model {e_emu}")
            base_kv[0].append((k0[:, :PROMPT - 1].clone(), v0[:, :PROMPT - 1].clone()))
            base_kv[1].append((k1[:, :PROMPT - 1].clone(), v1[:, :PROMPT - 1].clone()))
            base_kv_emu.append((k0e[:, :PROMPT - 1].clone(), v0e[:, :PROMPT - 1].clone()))
        del x0, x0e, x1
        t_prefill = time.time() - t_start

        # ---- oracle: every decode module, teacher-forced on the GPU tokens ----
        logit = {"gpu": {}, "emu": {}}
        flips, flips_emu, margins_at_flip, n_tok = 0, 0, [], 0
        for m in range(N_MOD):
            mod = eng.mods[m]
            emb = mod.embed.cpu().float()
            xs = []
            for s in range(2):
                feed = [int(prompts[s][-1])] + [int(t) for t in toks[s, m, :MAX_NEW - 1]]
                xs.append(emb[torch.tensor(feed, dtype=torch.long)])
            xe = xs[0].clone()
            del emb
            for l in range(cfg.n_layers):
                lw = mod.layer_reference(l)
                for s in range(2):
                    xs[s], _ = layer_forward(cfg, lw, xs[s], base_kv[s][l], cos, sin)
                xe, _ = layer_forward(cfg, lw, xe, base_kv_emu[l], cos, sin, bf16_storage=True)
                del lw
            fn, head = mod.final_norm.cpu().float(), mod.head.cpu().float()
            lge = final_logits(cfg, fn, head, xe, bf16_storage=True)
            for s in range(2):
                lg = final_logits(cfg, fn, head, xs[s])  # [MAX_NEW, vocab]
                row = inv[s * N_MOD + m]
                for key, got, want, emu in (("first", first_gpu[row], lg[0], lge[0]),
                                            ("last", last_gpu[row], lg[-1], lge[-1])):
                    e = _rel(got, want)
                    logit["gpu"][f"m{m}s{s}_{key}"] = [round(x, 5) for x in e]
                    if s == 0:
                        logit["emu"][f"m{m}s0_{key}"] = [round(x, 5) for x in _rel(emu, want)]
                    ee = _rel(lge[0 if key == "first" else -1], lg[0 if key == "first" else -1]) if s == 0 else \
                        tuple(max(v[i] for k2, v in logit["emu"].items() if k2.endswith(key)) for i in range(2))
                    if not (e[1] <= LOGIT_K * ee[1] + 5e-3 and e[0] <= LOGIT_K * ee[0] + 1e-2):
                        fails.append(f"module {m} session {s} {key} logits err (max, fro) {e} vs bf16 model {ee}")
                top2 = torch.topk(lg, 2, dim=-1).values
                marg = (top2[:, 0] - top2[:, 1])
                scale = lg.abs().max(dim=-1).values
                want_tok = lg.argmax(dim=-1).numpy()
                got_tok = toks[s, m]
                for t in np.nonzero(want_tok != got_tok)[0]:
                    flips += 1
                    margins_at_flip.append(float(marg[t] / scale[t]))
                    if not marg[t] <= TIE_RTOL * scale[t]:
                        fails.append(f"module {m} session {s} step {t}: token {got_tok[t]} != {want_tok[t]}, "
                                     f"margin {float(marg[t])}")
                if s == 0:
                    flips_emu += int((lge.argmax(dim=-1).numpy() != want_tok).sum())
                n_tok += MAX_NEW
            del head
    report = {"config": "8B shape, 32 layers, 2 x 4096-token prompts (2048 shared), 4 modules, 256 tokens, "
                        "32 rows/module (K5-TC)",
              "kv_gpu_vs_fp32_max_fro": kv["gpu"], "kv_bf16model_vs_fp32_max_fro": kv["emu"],
              "kv_gpu_vs_bf16model_max_fro": kv["gpu_vs_emu"], "kv_session1_gpu_vs_fp32_max_fro": kv["gpu_s1"],
              "logits_gpu_vs_fp32_max_fro": logit["gpu"], "logits_bf16model_vs_fp32_max_fro": logit["emu"],
              "tokens_checked": n_tok, "flips_gpu_vs_fp32": flips,
              "flips_bf16model_vs_fp32_session0": flips_emu, "tokens_session0": n_tok // 2,
              "flip_margins_rel": [round(x, 5) for x in margins_at_flip],
              "oracle_prefill_s": round(t_prefill, 1), "total_s": round(time.time() - t_start, 1),
              "failures": fails[:20]}
    print(json.dumps(report))
    out = os.environ.get("PSK_PARITY_OUT")
    if out:
        os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
        with open(out, "w") as f:
            json.dump(report, f, indent=1)
    assert not fails, fails[:10]
    # greedy flips only at near-ties, and no more often than bf16 storage
    # itself flips them (random-init logits are nearly flat)
    assert flips <= 2 * FLIP_K * flips_emu + 16
