"""Literal CPU restatement of the reference TinyLM — TEST INFRASTRUCTURE ONLY.

Follows frontend/src/rng.ts:9-82 (splitmix64, mixSeed, Rng) and
frontend/src/model.ts (LayerNorm eps 1e-5 with biased variance :120-123,
GELU-tanh :114-118, parameter order and init :139-198, forward :246-331,
PromptCache slice/row :41-88, buildBaseCache :340-352, generate :363-412)
and frontend/src/evaluate.ts:16-50. fp32 via torch (tfjs is fp32).

Parity status: UNPINNED at the tensor level — node/tfjs are absent from the
image and the reference publishes no tensor golden values; rng.test.ts seed-0
vectors pin the RNG, and the reference's KV-cache property tests
(model.test.ts:79-191, A9) are mirrored in tests/test_oracle_tinylm.py.
The B200 kernels implement the Llama-style modules (oracle/model.py); this
module exists to check the prefill/decode factorisation semantics the
reference defines.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

M64 = (1 << 64) - 1


def splitmix64(state: int) -> tuple[int, int]:
    """rng.ts:9-16: returns (next_state, output)."""
    s = (state + 0x9E3779B97F4A7C15) & M64
    z = s
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return s, (z ^ (z >> 31)) & M64


def mix_seed(master: int, *labels) -> int:
    """rng.ts:19-36 (string labels hash char codes plus a length marker)."""
    state = master & M64
    for label in labels:
        if isinstance(label, str):
            parts = [ord(c) for c in label] + [0x100000000 + len(label)]
        else:
            parts = [int(label) & M64]
        for p in parts:
            _, state = splitmix64((state ^ p) & M64)
    return state


class Rng:
    """rng.ts:39-82."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def next_u64(self) -> int:
        self.state, z = splitmix64(self.state)
        return z

    def float(self) -> float:
        return (self.next_u64() >> 11) / 2.0 ** 53

    def int(self, n: int) -> int:
        if n <= 0:
            raise ValueError(f"int() requires n > 0, got {n}")
        return math.floor(self.float() * n)

    def gauss(self) -> float:
        u1 = 1 - self.float()
        u2 = self.float()
        return math.sqrt(-2 * math.log(u1)) * math.cos(2 * math.pi * u2)


@dataclass(frozen=True)
class TinyConfig:
    layers: int
    width: int
    heads: int
    context: int
    vocab: int


class PromptCache:
    """model.ts:41-88: per-layer K/V [B, H, S, hd] + covered token ids."""

    def __init__(self, layers, tokens):
        self.layers = layers
        self.tokens = [list(t) for t in tokens]
        self.batch = len(tokens)
        self.length = len(tokens[0]) if tokens else 0

    def slice(self, n: int) -> "PromptCache":
        if n < 0 or n > self.length:
            raise ValueError(f"slice length {n} outside [0, {self.length}]")
        return PromptCache([(k[:, :, :n], v[:, :, :n]) for k, v in self.layers],
                           [t[:n] for t in self.tokens])

    def row(self, b: int) -> "PromptCache":
        if b < 0 or b >= self.batch:
            raise ValueError(f"row {b} outside [0, {self.batch})")
        return PromptCache([(k[b:b + 1], v[b:b + 1]) for k, v in self.layers], [self.tokens[b]])


def _gelu(x):
    return 0.5 * x * (1 + torch.tanh((x + 0.044715 * x * x * x) * math.sqrt(2 / math.pi)))


def _ln(x, g, b):
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)  # tf.moments: biased variance
    return (x - mean) / torch.sqrt(var + 1e-5) * g + b


class TinyLM:
    def __init__(self, cfg: TinyConfig, params: dict):
        if cfg.width % cfg.heads:
            raise ValueError(f"width {cfg.width} not divisible by heads {cfg.heads}")
        self.cfg = cfg
        self.p = params

    @staticmethod
    def init(cfg: TinyConfig, seed: int) -> "TinyLM":
        """model.ts:181-198 — parameters drawn in variables() order (:200-207)."""
        if cfg.width % cfg.heads:
            raise ValueError(f"width {cfg.width} not divisible by heads {cfg.heads}")
        rng = Rng(seed)
        d = cfg.width

        def init(*shape):
            n = math.prod(shape)
            return torch.tensor([0.02 * rng.gauss() for _ in range(n)], dtype=torch.float32).view(*shape)

        # construction order of model.ts:147-169
        p = {"tokEmb": init(cfg.vocab, d), "prevEmb": init(cfg.vocab, d), "posEmb": init(cfg.context, d),
             "blocks": []}
        for _ in range(cfg.layers):
            p["blocks"].append({
                "ln1g": torch.ones(d), "ln1b": torch.zeros(d),
                "wq": init(d, d), "wk": init(d, d), "wv": init(d, d), "wo": init(d, d),
                "ln2g": torch.ones(d), "ln2b": torch.zeros(d),
                "wUp": init(d, 4 * d), "bUp": torch.zeros(4 * d),
                "wDown": init(4 * d, d), "bDown": torch.zeros(d),
            })
        p["lnFg"], p["lnFb"] = torch.ones(d), torch.zeros(d)
        p["head"] = init(d, cfg.vocab)
        eye = torch.eye(d) * 0.5
        for b in p["blocks"]:
            b["wq"] = b["wq"] + eye
            b["wk"] = b["wk"] + eye
        p["prevEmb"] = p["prevEmb"] * 0.25 + p["tokEmb"]
        return TinyLM(cfg, p)

    def forward(self, tokens, past: PromptCache | None = None):
        """model.ts:246-331."""
        B, T = len(tokens), len(tokens[0])
        if any(len(r) != T for r in tokens):
            raise ValueError("ragged token batch")
        S0 = past.length if past else 0
        if past is not None and past.batch != B:
            raise ValueError(f"cache batch {past.batch} != token batch {B}")
        if S0 + T > self.cfg.context:
            raise ValueError(f"sequence length {S0 + T} exceeds context {self.cfg.context}")
        d, H = self.cfg.width, self.cfg.heads
        hd = d // H
        p = self.p
        prev = [[(tokens[b][i - 1] if i > 0 else (past.tokens[b][S0 - 1] if past else -1))
                 for i in range(T)] for b in range(B)]
        ids = torch.tensor(tokens)
        pid = torch.tensor(prev)
        x = p["tokEmb"][ids] + torch.where((pid >= 0)[..., None], p["prevEmb"][pid.clamp(min=0)],
                                           torch.zeros(d))
        x = x + p["posEmb"][S0:S0 + T][None]
        S = S0 + T
        mask = torch.where(torch.arange(S)[None, :] <= (S0 + torch.arange(T))[:, None], 0.0, -1e9)
        out_layers = []
        for l, bw in enumerate(p["blocks"]):
            xn = _ln(x, bw["ln1g"], bw["ln1b"])
            split = lambda w: (xn.reshape(B * T, d) @ w).view(B, T, H, hd).transpose(1, 2)  # noqa: E731
            q, k, v = split(bw["wq"]), split(bw["wk"]), split(bw["wv"])
            if past is not None:
                k = torch.cat([past.layers[l][0], k], 2)
                v = torch.cat([past.layers[l][1], v], 2)
            out_layers.append((k, v))
            att = torch.softmax(q @ k.transpose(2, 3) / math.sqrt(hd) + mask, -1)
            ctx = (att @ v).transpose(1, 2).reshape(B * T, d)
            x = x + (ctx @ bw["wo"]).view(B, T, d)
            xm = _ln(x, bw["ln2g"], bw["ln2b"])
            h = _gelu(xm.reshape(B * T, d) @ bw["wUp"] + bw["bUp"])
            x = x + (h @ bw["wDown"] + bw["bDown"]).view(B, T, d)
        logits = (_ln(x, p["lnFg"], p["lnFb"]).reshape(B * T, d) @ p["head"]).view(B, T, -1)
        covered = [(past.tokens[b] if past else []) + list(tokens[b]) for b in range(B)]
        return logits, PromptCache(out_layers, covered)


def build_base_cache(base: TinyLM, prompts) -> PromptCache:
    """model.ts:340-352."""
    if len(prompts[0]) > base.cfg.context:
        raise ValueError("prompt length exceeds context")
    with torch.no_grad():
        return base.forward(prompts)[1]


def generate(model: TinyLM, prompt, max_new: int, incremental: bool = True, past=None) -> list[int]:
    """model.ts:363-412."""
    if past is not None and past.batch != 1:
        raise ValueError("generate() takes a batch-1 cache")
    if past is not None and past.length >= len(prompt):
        raise ValueError("injected cache must cover a strict prefix of the prompt")
    out: list[int] = []
    if max_new <= 0:
        return out
    with torch.no_grad():
        if incremental:
            fresh = list(prompt[past.length if past else 0:])
            logits, cache = model.forward([fresh], past)
            nxt = int(torch.argmax(logits[0, -1]))
            for t in range(max_new):
                out.append(nxt)
                if t == max_new - 1:
                    break
                logits, cache = model.forward([[out[-1]]], cache)
                nxt = int(torch.argmax(logits[0, -1]))
        else:
            for _ in range(max_new):
                logits, _ = model.forward([list(prompt) + out])
                out.append(int(torch.argmax(logits[0, -1])))
    return out


def shared_prefix_length(ratio: float, n: int) -> int:
    """evaluate.ts:16-19."""
    if not (0 <= ratio <= 1):
        raise ValueError(f"sharing ratio {ratio} outside [0, 1]")
    return min(math.ceil(ratio * n), n - 1)


def evaluate_sharing_predictions(dec: TinyLM, base: TinyLM, ratio: float, prompts) -> list[int]:
    """evaluate.ts:21-50 (returns the greedy predictions instead of accuracy)."""
    if not prompts:
        raise ValueError("empty evaluation set")
    n = len(prompts[0])
    if any(len(p) != n for p in prompts):
        raise ValueError("evaluation prompts must share a length")
    m = shared_prefix_length(ratio, n)
    with torch.no_grad():
        past = build_base_cache(base, prompts).slice(m) if m > 0 else None
        logits, _ = dec.forward([p[m:] for p in prompts], past)
    return torch.argmax(logits[:, -1], -1).tolist()
