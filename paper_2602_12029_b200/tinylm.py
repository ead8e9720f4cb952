"""The reference's TinyLM (frontend/src/model.ts, rng.ts, evaluate.ts) on the
GPU: fp32 forward in one kernel per call (psk_tiny_forward, csrc/tinylm.cu)
over a paged prompt cache.

API as the reference (names in snake_case; RangeError -> ValueError):
  TinyLM.init(cfg, seed)                     model.ts:139-198 (+ rng.ts init)
  TinyLM.forward(tokens, past) -> (logits, cache)   model.ts:246-331
  PromptCache.slice(n) / .row(b)             model.ts:58-88
  build_base_cache(base, prompts)            model.ts:340-352
  generate(model, prompt, max_new, incremental, past)   model.ts:363-412
  shared_prefix_length / evaluate_sharing    evaluate.ts:16-50

The prompt cache is a set of 16-token pages in a TinyKVPool plus a block
table per row, instead of model.ts's concatenated [B, H, S, hd] tensors:
slice(n) keeps the first ceil(n / 16) pages, so a decode module's forward on
a base cache reads the base's pages in place and appends to its own. Pages
are append-only with a fill mark: a forward that would write into a page
someone else already filled past its start position copies that page
first (copy-on-write of the one partial page at the slice point).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

PAGE = 16
M64 = (1 << 64) - 1
_LAYER_KEYS = ("ln1g", "ln1b", "wq", "wk", "wv", "wo", "ln2g", "ln2b", "wUp", "bUp", "wDown", "bDown")


def splitmix64(state: int) -> tuple[int, int]:
    """rng.ts:9-16: (next state, output)."""
    s = (state + 0x9E3779B97F4A7C15) & M64
    z = ((s ^ (s >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return s, (z ^ (z >> 31)) & M64


class Rng:
    """rng.ts:39-82 (the uniform / Box-Muller draws the init uses)."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def float(self) -> float:
        self.state, z = splitmix64(self.state)
        return (z >> 11) / 2.0 ** 53

    def gauss(self) -> float:
        u1 = 1 - self.float()
        u2 = self.float()
        return math.sqrt(-2 * math.log(u1)) * math.cos(2 * math.pi * u2)


@dataclass(frozen=True)
class TinyConfig:
    """model.ts:17-31 (DEFAULT_MODEL: 4 layers, width 128, 4 heads, context 256)."""
    layers: int = 4
    width: int = 128
    heads: int = 4
    context: int = 256
    vocab: int = 64


class TinyKVPool:
    """Pages [page][layer][K|V][head][16][hd] fp32 on one GPU, handed out in
    order and never reused (size it for the caches a run builds; models
    that share one pool read each other's caches in place); `filled[p]` =
    tokens written into page p so far (append-only)."""

    def __init__(self, cfg: TinyConfig, n_pages: int, device: int = 0):
        hd = cfg.width // cfg.heads
        self.cfg = cfg
        self.data = torch.zeros(n_pages, cfg.layers, 2, cfg.heads, PAGE, hd, dtype=torch.float32,
                                device=torch.device("cuda", device))
        self.filled = np.zeros(n_pages, dtype=np.int64)
        self.next = 0

    def alloc(self) -> int:
        if self.next >= self.data.shape[0]:
            raise RuntimeError(f"TinyKVPool: all {self.data.shape[0]} pages in use")
        self.next += 1
        return self.next - 1


class PromptCache:
    """model.ts:41-88: per-row block tables into a TinyKVPool plus the covered
    token ids (the prev-token channel needs the last one, model.ts:270)."""

    def __init__(self, pool: TinyKVPool, tables, tokens):
        self.pool = pool
        self.tables = [list(t) for t in tables]
        self.tokens = [list(t) for t in tokens]
        self.batch = len(self.tokens)
        self.length = len(self.tokens[0]) if self.tokens else 0

    def slice(self, n: int) -> "PromptCache":
        """model.ts:58-70: the first n positions (no copy: a shorter table)."""
        if n < 0 or n > self.length:
            raise ValueError(f"slice length {n} outside [0, {self.length}]")
        keep = (n + PAGE - 1) // PAGE
        return PromptCache(self.pool, [t[:keep] for t in self.tables], [t[:n] for t in self.tokens])

    def row(self, b: int) -> "PromptCache":
        """model.ts:72-88."""
        if b < 0 or b >= self.batch:
            raise ValueError(f"row {b} outside [0, {self.batch})")
        return PromptCache(self.pool, [self.tables[b]], [self.tokens[b]])

    def kv(self, layer: int, row: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
        """K, V of one row and layer as [H, S, hd] (model.ts's layout), for tests."""
        pages = self.pool.data[torch.tensor(self.tables[row], dtype=torch.long, device=self.pool.data.device)]
        kvl = pages[:, layer]  # [P, 2, H, 16, hd]
        H, hd = kvl.shape[2], kvl.shape[4]
        flat = kvl.permute(1, 2, 0, 3, 4).reshape(2, H, -1, hd)[:, :, :self.length]
        return flat[0], flat[1]


def init_params(cfg: TinyConfig, seed: int) -> dict:
    """model.ts:181-198 on the host: Gaussian(0, 0.02) draws (rng.ts) in
    construction order (:147-169), LayerNorm gains 1 / biases 0, 0.5 I added
    to wq / wk, prevEmb = 0.25 prevEmb + tokEmb."""
    if cfg.width % cfg.heads:
        raise ValueError(f"width {cfg.width} not divisible by heads {cfg.heads}")
    rng = Rng(seed)
    d = cfg.width

    def init(*shape):
        n = math.prod(shape)
        return torch.tensor([0.02 * rng.gauss() for _ in range(n)], dtype=torch.float32).view(*shape)

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
    return p


class TinyLM:
    """model.ts:112-331 with its weights on the GPU (fp32)."""

    def __init__(self, cfg: TinyConfig, params: dict, device: int = 0, pool: TinyKVPool | None = None,
                 pool_pages: int | None = None):
        if cfg.width % cfg.heads:
            raise ValueError(f"width {cfg.width} not divisible by heads {cfg.heads}")
        self.cfg = cfg
        self.dev = torch.device("cuda", device)
        to = lambda t: t.to(self.dev, torch.float32).contiguous()  # noqa: E731
        self.p = {k: to(params[k]) for k in ("tokEmb", "prevEmb", "posEmb", "lnFg", "lnFb", "head")}
        self.p["blocks"] = [{k: to(b[k]) for k in _LAYER_KEYS} for b in params["blocks"]]
        ptrs = [b[k].data_ptr() for b in self.p["blocks"] for k in _LAYER_KEYS]
        self._ptrs = torch.tensor(ptrs, dtype=torch.int64, device=self.dev)
        self._c = _lib.TinyModelC(cfg.layers, cfg.width, cfg.heads, cfg.context, cfg.vocab,
                                  self.p["tokEmb"].data_ptr(), self.p["prevEmb"].data_ptr(),
                                  self.p["posEmb"].data_ptr(), self.p["lnFg"].data_ptr(),
                                  self.p["lnFb"].data_ptr(), self.p["head"].data_ptr(), self._ptrs.data_ptr())
        self.pool = pool or TinyKVPool(cfg, pool_pages or 4096, device)
        self._lib = _lib.load()

    @staticmethod
    def init(cfg: TinyConfig, seed: int, **kw) -> "TinyLM":
        """model.ts:181-198 (parameters from init_params), on the GPU."""
        return TinyLM(cfg, init_params(cfg, seed), **kw)

    def _import(self, past: PromptCache) -> PromptCache:
        """A cache built by a model with another page pool (model.ts caches
        are plain tensors any model can consume): its pages copied into this
        model's pool (same layer / head geometry required)."""
        if past.pool.data.shape[1:] != self.pool.data.shape[1:]:
            raise ValueError("cache geometry (layers, heads, head dim) differs from this model's")
        tables = []
        for t in past.tables:
            new = [self.pool.alloc() for _ in t]
            if new:
                src = torch.tensor(t, dtype=torch.long, device=past.pool.data.device)
                dst = torch.tensor(new, dtype=torch.long, device=self.dev)
                self.pool.data[dst] = past.pool.data[src].to(self.dev)
                self.pool.filled[new] = past.pool.filled[t]
            tables.append(new)
        return PromptCache(self.pool, tables, past.tokens)

    def _writable_table(self, table: list[int], s0: int, n_new: int) -> list[int]:
        """Pages for positions s0 .. s0 + n_new - 1 appended to a row's table;
        a partially filled last page that someone else has filled past s0 is
        copied first (copy-on-write)."""
        pool, t = self.pool, list(table)
        if s0 % PAGE and pool.filled[t[s0 // PAGE]] != s0 % PAGE:
            src, dst = t[s0 // PAGE], pool.alloc()
            pool.data[dst].copy_(pool.data[src])
            pool.filled[dst] = s0 % PAGE
            t[s0 // PAGE] = dst
        while len(t) * PAGE < s0 + n_new:
            t.append(pool.alloc())
        return t

    def forward(self, tokens, past: PromptCache | None = None):
        """model.ts:246-331 -> (logits [B, T, vocab] fp32 on the GPU, cache)."""
        B = len(tokens)
        if B == 0:
            raise ValueError("empty token batch")
        T = len(tokens[0])
        if T == 0 or any(len(r) != T for r in tokens):
            raise ValueError("ragged token batch")
        if past is not None and past.batch != B:
            raise ValueError(f"cache batch {past.batch} != token batch {B}")
        s0 = past.length if past is not None else 0
        if s0 + T > self.cfg.context:
            raise ValueError(f"sequence length {s0 + T} exceeds context {self.cfg.context}")
        if past is not None and past.pool is not self.pool:
            past = self._import(past)
        tables = [self._writable_table(past.tables[b] if past is not None else [], s0, T) for b in range(B)]
        maxp = max(len(t) for t in tables)
        tab = np.array([t + [t[0]] * (maxp - len(t)) for t in tables], dtype=np.int32)
        prev = np.array([past.tokens[b][-1] if past is not None and s0 > 0 else -1 for b in range(B)],
                        dtype=np.int32)
        host = np.asarray(tokens, dtype=np.int64)
        if host.min() < 0 or host.max() >= self.cfg.vocab:  # checked on the host: no device sync
            raise ValueError("token id outside the vocabulary")
        toks = torch.from_numpy(host.astype(np.int32)).to(self.dev)
        d_tab = torch.from_numpy(tab).to(self.dev)
        d_prev = torch.from_numpy(prev).to(self.dev)
        nf = C.c_int64()
        _lib.check(self._lib.psk_tiny_scratch_floats(C.byref(self._c), B, T, C.byref(nf)))
        scratch = torch.empty(nf.value, dtype=torch.float32, device=self.dev)
        logits = torch.empty(B, T, self.cfg.vocab, dtype=torch.float32, device=self.dev)
        _lib.check(self._lib.psk_tiny_forward(
            C.byref(self._c), B, T, s0, toks.data_ptr(), d_prev.data_ptr(), d_tab.data_ptr(), maxp,
            self.pool.data.data_ptr(), self.pool.data.shape[0], scratch.data_ptr(), logits.data_ptr(),
            torch.cuda.current_stream(self.dev).cuda_stream))
        for t in tables:  # fill marks of the pages written
            for i in range(s0 // PAGE, (s0 + T - 1) // PAGE + 1):
                self.pool.filled[t[i]] = max(self.pool.filled[t[i]], min(PAGE, s0 + T - i * PAGE))
        covered = [(past.tokens[b] if past is not None else []) + list(tokens[b]) for b in range(B)]
        return logits, PromptCache(self.pool, tables, covered)


def build_base_cache(base: TinyLM, prompts) -> PromptCache:
    """model.ts:340-352: the frozen base module's forward over the prompts."""
    if len(prompts[0]) > base.cfg.context:
        raise ValueError("prompt length exceeds context")
    return base.forward(prompts)[1]


def generate(model: TinyLM, prompt, max_new: int, incremental: bool = True, past=None) -> list[int]:
    """model.ts:363-412: greedy; incremental from an injected strict-prefix cache."""
    if past is not None and past.batch != 1:
        raise ValueError("generate() takes a batch-1 cache")
    if past is not None and past.length >= len(prompt):
        raise ValueError("injected cache must cover a strict prefix of the prompt")
    out: list[int] = []
    if max_new <= 0:
        return out
    if incremental:
        logits, cache = model.forward([list(prompt[past.length if past is not None else 0:])], past)
        nxt = int(torch.argmax(logits[0, -1]))
        for t in range(max_new):
            out.append(nxt)
            if t == max_new - 1:
                break
            logits, cache = model.forward([[nxt]], cache)
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


def sharing_predictions(dec: TinyLM, base: TinyLM, ratio: float, prompts) -> list[int]:
    """evaluate.ts:21-43: the decode module's greedy prediction after the
    base's cache of the first m positions."""
    if not prompts:
        raise ValueError("empty evaluation set")
    n = len(prompts[0])
    if any(len(p) != n for p in prompts):
        raise ValueError("evaluation prompts must share a length")
    m = shared_prefix_length(ratio, n)
    past = build_base_cache(base, prompts).slice(m) if m > 0 else None
    logits, _ = dec.forward([list(p[m:]) for p in prompts], past)
    return torch.argmax(logits[:, -1], -1).tolist()


def evaluate_sharing(dec: TinyLM, base: TinyLM, ratio: float, eval_set) -> float:
    """evaluate.ts:21-50: exact-match accuracy over (prompt, target) samples."""
    if not eval_set:
        raise ValueError("empty evaluation set")
    preds = sharing_predictions(dec, base, ratio, [s[0] for s in eval_set])
    return sum(int(p == s[1]) for p, s in zip(preds, eval_set)) / len(eval_set)
