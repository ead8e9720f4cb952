"""Accuracy under partial KV-cache sharing on the GPU path
(frontend/src/evaluate.ts:16-50).

At sharing ratio r the first m = min(ceil(r n), n - 1) prompt positions'
keys/values come from the frozen base module's cache (buildBaseCache,
model.ts:340-352); the evaluated decode module recomputes positions
[m, n) on top of it (its forward with `past`, model.ts:246-331) and its
last-position logits give the greedy prediction; scoring is exact match.
Here: the base module's batched prefill of [0, m) writes the paged cache,
the decode module's batched prefill of [m, n) continues in the same pages
(K1-K3 with the decode module's weights), then final RMSNorm + LM head
(K5 GEMV) + argmax on the last rows.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .model import PAGE_TOKENS, KVCache, LlamaConfig, ModuleWeights, PrefillRunner, _ptr, _stream


def shared_prefix_length(ratio: float, prompt_len: int) -> int:
    """evaluate.ts:16-19."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError(f"sharing ratio {ratio} outside [0, 1]")  # RangeError in the reference
    return min(math.ceil(ratio * prompt_len), prompt_len - 1)


class SharingEvaluator:
    """Reusable buffers for evaluate_sharing at one (config, batch, length)."""

    def __init__(self, cfg: LlamaConfig, max_prompts: int, prompt_len: int, device: int = 0):
        self.cfg, self.n = cfg, prompt_len
        self.pages_per = (prompt_len + PAGE_TOKENS - 1) // PAGE_TOKENS
        self.kv = KVCache(cfg, max_prompts * self.pages_per, device)
        self.dev = torch.device("cuda", device)
        self.max_prompts = max_prompts
        self.lib = _lib.load()
        f32 = torch.float32
        self.xn = torch.empty(max_prompts, cfg.d_model, dtype=torch.bfloat16, device=self.dev)
        self.logits = torch.empty(max_prompts, cfg.vocab, dtype=f32, device=self.dev)
        self.pred = torch.empty(max_prompts, dtype=torch.int32, device=self.dev)
        self.mrs = torch.tensor([0, 0], dtype=torch.int32, device=self.dev)

    def predictions(self, dec: ModuleWeights, base: ModuleWeights, ratio: float, prompts) -> np.ndarray:
        cfg, lib = self.cfg, self.lib
        B = len(prompts)
        if B == 0:
            raise ValueError("empty evaluation set")
        if B > self.max_prompts or any(len(p) != self.n for p in prompts):
            raise ValueError("evaluation prompts must share the evaluator's length")  # RangeError in the reference
        m = shared_prefix_length(ratio, self.n)
        toks = [torch.as_tensor(np.asarray(p, dtype=np.int64), device=self.dev) for p in prompts]
        tables = [list(range(i * self.pages_per, (i + 1) * self.pages_per)) for i in range(B)]
        T = self.n - m
        if m > 0:
            PrefillRunner(cfg, base, self.kv, max_tokens=B * m).run_batch(
                [(t[:m], 0, pt) for t, pt in zip(toks, tables)], kv_only=True)
        runner = PrefillRunner(cfg, dec, self.kv, max_tokens=B * T)
        runner.run_batch([(t[m:], m, pt) for t, pt in zip(toks, tables)])
        s = _stream()
        last = torch.arange(B, device=self.dev) * T + (T - 1)  # each sequence's last position
        h_last = runner.h[last].contiguous()
        g = torch.tensor([dec.final_norm.data_ptr()], dtype=torch.int64, device=self.dev)
        _lib.check(lib.psk_rmsnorm_rows(_ptr(h_last), B, cfg.d_model, _ptr(g), None, float(cfg.norm_eps),
                                        _ptr(self.xn), s))
        head = torch.tensor([dec.head.data_ptr()], dtype=torch.int64, device=self.dev)
        for r0 in range(0, B, 32):  # K5: <= 32 rows per module per launch
            nr = min(32, B - r0)
            self.mrs[1] = nr
            _lib.check(lib.psk_gemv(_ptr(self.xn[r0:]), nr, cfg.d_model, _ptr(head), _ptr(self.mrs), 1, nr,
                                    cfg.vocab, 1, _ptr(self.logits[r0:]), s))
        _lib.check(lib.psk_argmax_rows(_ptr(self.logits), B, cfg.vocab, _ptr(self.pred), s))
        return self.pred[:B].cpu().numpy()


def evaluate_sharing(dec: ModuleWeights, base: ModuleWeights, ratio: float, prompts, targets,
                     evaluator: SharingEvaluator | None = None) -> float:
    """evaluate.ts:21-50: exact-match accuracy of `dec` when the first
    shared_prefix_length(ratio, n) positions come from `base`'s cache."""
    if len(prompts) == 0:
        raise ValueError("empty evaluation set")
    ev = evaluator or SharingEvaluator(dec.cfg, len(prompts), len(prompts[0]), dec.embed.device.index or 0)
    pred = ev.predictions(dec, base, ratio, prompts)
    return float(np.mean(pred == np.asarray(targets)))
