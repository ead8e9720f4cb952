"""Pin the Llama oracle against an independent implementation.

Runs transformers' LlamaForCausalLM (installed in this image) on weights
drawn from numpy's PCG64 (seed below; reproducible everywhere, so the test
regenerates them) and stores its logits, greedy continuation and KV cache
for a short prompt in tests/golden/llama_tiny.npz. The test feeds the same
weights to oracle.model.LlamaOracle and must match within fp32 tolerance.

    python tests/golden/make_llama_golden.py
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "llama_tiny.npz"
SEED = 20260212
CFG = dict(n_layers=2, d_model=256, n_heads=2, n_kv_heads=1, ffn=768, vocab=512,
           rope_theta=10000.0, norm_eps=1e-5, head_dim=128, max_pos=256)
PROMPT = [int(x) for x in np.random.default_rng(7).integers(0, 512, size=24)]
MAX_NEW = 12


def make_weights(cfg=CFG, seed=SEED) -> dict:
    """Standard-layout fp32 weights (numpy), shared by this script and the test."""
    rng = np.random.default_rng(seed)
    d, f, hd = cfg["d_model"], cfg["ffn"], cfg["head_dim"]
    n = lambda *s: (0.02 * rng.standard_normal(s)).astype(np.float32)  # noqa: E731
    g = lambda: (1.0 + 0.1 * rng.standard_normal(d)).astype(np.float32)  # noqa: E731
    w = {"embed": n(cfg["vocab"], d), "layers": []}
    for _ in range(cfg["n_layers"]):
        w["layers"].append({
            "attn_norm": g(), "wq": n(cfg["n_heads"] * hd, d), "wk": n(cfg["n_kv_heads"] * hd, d),
            "wv": n(cfg["n_kv_heads"] * hd, d), "wo": n(d, cfg["n_heads"] * hd), "mlp_norm": g(),
            "w_gate": n(f, d), "w_up": n(f, d), "w_down": n(d, f),
        })
    w["final_norm"] = g()
    w["head"] = n(cfg["vocab"], d)
    return w


def main() -> None:
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    w = make_weights()
    hc = LlamaConfig(vocab_size=CFG["vocab"], hidden_size=CFG["d_model"],
                     intermediate_size=CFG["ffn"], num_hidden_layers=CFG["n_layers"],
                     num_attention_heads=CFG["n_heads"], num_key_value_heads=CFG["n_kv_heads"],
                     head_dim=CFG["head_dim"], rms_norm_eps=CFG["norm_eps"],
                     rope_theta=CFG["rope_theta"], max_position_embeddings=CFG["max_pos"],
                     tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    m = LlamaForCausalLM(hc).eval().float()
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"],
          "lm_head.weight": w["head"]}
    for i, lw in enumerate(w["layers"]):
        p = f"model.layers.{i}."
        sd.update({p + "input_layernorm.weight": lw["attn_norm"],
                   p + "self_attn.q_proj.weight": lw["wq"], p + "self_attn.k_proj.weight": lw["wk"],
                   p + "self_attn.v_proj.weight": lw["wv"], p + "self_attn.o_proj.weight": lw["wo"],
                   p + "post_attention_layernorm.weight": lw["mlp_norm"],
                   p + "mlp.gate_proj.weight": lw["w_gate"], p + "mlp.up_proj.weight": lw["w_up"],
                   p + "mlp.down_proj.weight": lw["w_down"]})
    m.load_state_dict({k: torch.from_numpy(v) for k, v in sd.items()}, strict=True)
    ids = torch.tensor([PROMPT])
    with torch.no_grad():
        out = m(ids, use_cache=True)
        logits = out.logits[0].numpy()
        kv = out.past_key_values
        k0, v0 = kv.layers[0].keys[0].numpy(), kv.layers[0].values[0].numpy()
        k1, v1 = kv.layers[1].keys[0].numpy(), kv.layers[1].values[0].numpy()
        gen = m.generate(ids, max_new_tokens=MAX_NEW, do_sample=False)[0, len(PROMPT):].numpy()
    np.savez_compressed(OUT, prompt=np.array(PROMPT), logits=logits, k0=k0, v0=v0, k1=k1, v1=v1,
                        greedy=gen)
    print(f"wrote {OUT}: logits {logits.shape}, greedy {gen.tolist()}")


if __name__ == "__main__":
    main()
