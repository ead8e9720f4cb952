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


def _bf(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).float()


def layer_forward(cfg, lw: dict, x: torch.Tensor, past, cos_t: torch.Tensor, sin_t: torch.Tensor,
                  bf16_storage: bool = False):
    """One decoder layer (model.ts:296-325, Llama-style): x [T, d] holds the
    new positions [S, S+T); past = (K, V) [n_kv, S, hd] or None. Returns
    (x after the layer, (K, V) covering [0, S+T)). Used whole-model by
    LlamaOracle.forward and layer by layer (weights streamed per layer) by
    the full-size parity tests.

    bf16_storage=True is the PRECISION MODEL of the same algorithm: every
    tensor the kernels store in bf16 is rounded to bf16 at that point (norm
    outputs, rotated q/k and v (the paged cache), softmax probabilities
    before P.V, the attention output, the SwiGLU activation), everything else
    fp32 with exact max-subtracted softmax. The full-size parity test runs it
    beside the fp32 chain: the GPU must stay within a small factor of the
    error that bf16 storage alone implies."""
    r = _bf if bf16_storage else (lambda t: t)  # noqa: E731
    T = x.shape[0]
    S = past[0].shape[1] if past is not None else 0
    hd, H, Hk = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    cos, sin = cos_t[S:S + T], sin_t[S:S + T]
    h = r(_rms(x, lw["attn_norm"], cfg.norm_eps))
    q = (h @ lw["wq"].T).view(T, H, hd).transpose(0, 1)
    k = (h @ lw["wk"].T).view(T, Hk, hd).transpose(0, 1)
    v = r((h @ lw["wv"].T).view(T, Hk, hd).transpose(0, 1))
    q, k = r(_rope(q, cos, sin)), r(_rope(k, cos, sin))
    if past is not None:
        k = torch.cat([past[0], k], dim=1)
        v = torch.cat([past[1], v], dim=1)
    # key j visible to new position i iff j <= S + i (model.ts:288-293)
    mask = torch.arange(S + T)[None, :] <= (S + torch.arange(T))[:, None]
    grp = H // Hk
    o = torch.empty(H, T, hd)
    for g in range(Hk):  # per KV head: no repeat_interleave copy of a long cache
        qg = q[g * grp:(g + 1) * grp]
        sc = (qg @ k[g].T) / math.sqrt(hd)
        sc = sc.masked_fill(~mask, float("-inf"))
        if bf16_storage:
            e = torch.exp(sc - sc.max(dim=-1, keepdim=True).values)
            o[g * grp:(g + 1) * grp] = (r(e) @ v[g]) / e.sum(dim=-1, keepdim=True)
        else:
            o[g * grp:(g + 1) * grp] = torch.softmax(sc, dim=-1) @ v[g]
    x = x + r(o.transpose(0, 1).reshape(T, H * hd)) @ lw["wo"].T
    h2 = r(_rms(x, lw["mlp_norm"], cfg.norm_eps))
    g_ = h2 @ lw["w_gate"].T
    u = h2 @ lw["w_up"].T
    x = x + r(torch.nn.functional.silu(g_) * u) @ lw["w_down"].T
    return x, (k, v)


def decode_layer_batched(cfg, lw: dict, x: torch.Tensor, k_past: torch.Tensor, v_past: torch.Tensor,
                         cos_t: torch.Tensor, sin_t: torch.Tensor):
    """One decoder layer for R decode rows at once (one new token each, all
    at position S = k_past.shape[2]), each row over its own past K/V
    [R, n_kv, S, hd]: the batched form of layer_forward(T=1) that a CPU
    serving loop would run (every module's weights read once per step for
    all of its rows). Returns (x [R, d], (k, v) [R, n_kv, 1, hd] of the new
    token)."""
    R = x.shape[0]
    S = k_past.shape[2]
    hd, H, Hk = cfg.head_dim, cfg.n_heads, cfg.n_kv_heads
    cos, sin = cos_t[S:S + 1], sin_t[S:S + 1]
    h = _rms(x, lw["attn_norm"], cfg.norm_eps)
    q = _rope((h @ lw["wq"].T).view(R, H, 1, hd), cos, sin)
    k = _rope((h @ lw["wk"].T).view(R, Hk, 1, hd), cos, sin)
    v = (h @ lw["wv"].T).view(R, Hk, 1, hd)
    grp = H // Hk
    qg = q.view(R, Hk, grp, hd)
    sc = torch.cat([qg @ k_past.transpose(2, 3), qg @ k.transpose(2, 3)], dim=3) / math.sqrt(hd)
    pr = torch.softmax(sc, dim=-1)
    o = pr[..., :S] @ v_past + pr[..., S:] @ v  # [R, Hk, grp, hd]
    x = x + o.reshape(R, H * hd) @ lw["wo"].T
    h2 = _rms(x, lw["mlp_norm"], cfg.norm_eps)
    x = x + (torch.nn.functional.silu(h2 @ lw["w_gate"].T) * (h2 @ lw["w_up"].T)) @ lw["w_down"].T
    return x, (k, v)


def final_logits(cfg, final_norm: torch.Tensor, head: torch.Tensor, x: torch.Tensor,
                 bf16_storage: bool = False) -> torch.Tensor:
    """Final RMSNorm -> LM head (model.ts:327-328)."""
    h = _rms(x, final_norm, cfg.norm_eps)
    return (_bf(h) if bf16_storage else h) @ head.T


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
        x = w["embed"][torch.tensor(tokens, dtype=torch.long)]
        cache = []
        for l, lw in enumerate(w["layers"]):
            x, kv = layer_forward(c, lw, x, past[l] if past else None, self.cos, self.sin)
            cache.append(kv)
        logits = None
        if with_logits:
            logits = final_logits(c, w["final_norm"], w["head"], x)
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
