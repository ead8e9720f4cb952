"""fp32 CPU oracle of the module forward — TEST INFRASTRUCTURE ONLY.

Llama restatement (arch="llama") of what the B200 kernels compute, on
contiguous tensors: RMSNorm -> q,k,v -> RoPE (rotate-half) -> causal GQA
attention over [past; new] -> o-proj + residual -> RMSNorm -> SwiGLU MLP +
residual; final RMSNorm -> LM head. Its control flow restates the
reference TinyLM forward / buildBaseCache / generate
(frontend/src/model.ts:246-331, :340-352, :363-412): positions continue
from the cache length (:283), new positions attend to the cache and causally
to themselves (:288-293), the cache is concatenated per layer (:307-311),
an injected cache must be a strict prefix (:372-374) and decoding is greedy
argmax (:386, :396).

Pinned against transformers' LlamaForCausalLM on identical weights
(tests/golden/llama_tiny.npz, tests/golden/make_llama_golden.py).
"""

from __future__ import annotations

import math

import numpy as np
import torch


def rope_cos_sin(max_pos: int, head_dim: int, theta: float) -> tuple[torch.Tensor, torch.Tensor]:
    half = head_dim // 2
    inv = 1.0 / (theta ** (np.arange(half, dtype=np.float64) * 2.0 / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return (torch.from_numpy(np.cos(ang).astype(np.float32)),
            torch.from_numpy(np.sin(ang).astype(np.float32)))


def _rms(x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    # x [H, T, hd]; cos/sin [T, hd/2]
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


class LlamaOracle:
    """weights: dict from ModuleWeights.reference_layout() (fp32 CPU)."""

    def __init__(self, cfg, weights: dict):
        self.cfg = cfg
        self.w = weights
        self.cos, self.sin = rope_cos_sin(cfg.max_pos, cfg.head_dim, cfg.rope_theta)

    def forward(self, tokens, past=None, with_logits: bool = True):
        """tokens: list[int] (new positions); past: list of (K, V) per layer,
        each [n_kv, S, hd], covering positions [0, S). Returns (logits [T, V]
        or None, new cache [(K, V)] covering [0, S+T))."""
        c, w = self.cfg, self.w
        T = len(tokens)
        S = past[0][0].shape[1] if past else 0
        if S + T > c.max_pos:
            raise ValueError(f"sequence length {S + T} exceeds max_pos {c.max_pos}")
        hd, H, Hk = c.head_dim, c.n_heads, c.n_kv_heads
        x = w["embed"][torch.tensor(tokens, dtype=torch.long)]
        cos, sin = self.cos[S:S + T], self.sin[S:S + T]
        # key j visible to new position i iff j <= S + i (model.ts:288-293)
        mask = torch.arange(S + T)[None, :] <= (S + torch.arange(T))[:, None]
        cache = []
        for l, lw in enumerate(w["layers"]):
            h = _rms(x, lw["attn_norm"], c.norm_eps)
            q = (h @ lw["wq"].T).view(T, H, hd).transpose(0, 1)
            k = (h @ lw["wk"].T).view(T, Hk, hd).transpose(0, 1)
            v = (h @ lw["wv"].T).view(T, Hk, hd).transpose(0, 1)
            q, k = _rope(q, cos, sin), _rope(k, cos, sin)
            if past:
                k = torch.cat([past[l][0], k], dim=1)
                v = torch.cat([past[l][1], v], dim=1)
            cache.append((k, v))
            kk = k.repeat_interleave(H // Hk, dim=0)
            vv = v.repeat_interleave(H // Hk, dim=0)
            sc = (q @ kk.transpose(1, 2)) / math.sqrt(hd)
            sc = sc.masked_fill(~mask, float("-inf"))
            o = torch.softmax(sc, dim=-1) @ vv
            x = x + o.transpose(0, 1).reshape(T, H * hd) @ lw["wo"].T
            h2 = _rms(x, lw["mlp_norm"], c.norm_eps)
            g = h2 @ lw["w_gate"].T
            u = h2 @ lw["w_up"].T
            x = x + (torch.nn.functional.silu(g) * u) @ lw["w_down"].T
        logits = None
        if with_logits:
            logits = _rms(x, w["final_norm"], c.norm_eps) @ w["head"].T
        return logits, cache

    def prefill(self, tokens):
        """buildBaseCache (model.ts:340-352): K/V for every prompt position."""
        return self.forward(tokens, None, with_logits=False)[1]

    def generate(self, prompt, max_new: int, past=None, teacher=None):
        """Greedy decode (model.ts:363-399). `past` (if given) must cover a
        strict prefix of prompt (model.ts:372-374). `teacher`: optional forced
        next-token sequence (teacher forcing) — outputs still report argmax.
        Returns (argmax tokens, per-step logits)."""
        S = past[0][0].shape[1] if past else 0
        if past is not None and S >= len(prompt):
            raise ValueError("injected cache must cover a strict prefix of the prompt")
        out, logits_all = [], []
        if max_new <= 0:
            return out, logits_all
        logits, cache = self.forward(list(prompt[S:]), past)
        for t in range(max_new):
            lg = logits[-1]
            logits_all.append(lg)
            nxt = int(torch.argmax(lg))
            out.append(nxt)
            if t == max_new - 1:
                break
            feed = teacher[t] if teacher is not None else nxt
            logits, cache = self.forward([feed], cache)
        return out, logits_all
