"""PrefillShare serving engine on one B200 (the public API the bench's e2e
leg drives).

A batch of sessions is served the way the reference fleet serves a request
(src/prefillsim/cluster.py:271-442), with real GPU work in place of the
cost-model durations:

  prefill start   pool.longest_prefix_match (pins)         cluster.py:322-337
  prefill         base module forwards the uncached tokens  costs.py:46 -> K1-K3
  prefill done    pool.insert + pin of the new blocks       cluster.py:339-357
  handoff         zero-copy on one GPU: the decode modules  costs.py:66 -> (K8
                  read the prefill pages in place           on multi-GPU)
  decode          N decode modules x S sessions, greedy,    cluster.py:414-442
                  one CUDA-graph step per token (K5, K6)    costs.py:56
  release         pins drop; blocks stay cached             cluster.py:404-412

KV memory: pages [0, P) are owned by the GPU BlockPool (record slot == page,
so prefix hits are real KV reuse); pages [P, P + S*(1 + M*priv)) are the
sessions' partial-tail pages and the decode modules' private pages.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .kvstore import SHARED_NS, BlockChain, BlockPool
from .model import (PAGE_TOKENS, DecodeBatch, DecodeRow, DecodeRunner, KVCache, LlamaConfig,
                    ModuleWeights, PrefillRunner, SessionSpec)


@dataclass
class ServeResult:
    tokens: np.ndarray          # [S, n_modules, max_new] greedy outputs
    matched: list[int]          # prefix-hit tokens per session
    prefill_tokens: list[int]   # tokens the base module actually forwarded


class PrefillShareEngine:
    def __init__(self, cfg: LlamaConfig, n_modules: int, max_sessions: int, max_prompt: int,
                 max_new: int, pool_pages: int, seed: int = 0, device: int = 0,
                 modules: list[ModuleWeights] | None = None, base: ModuleWeights | None = None,
                 prefill_group: int = 2):
        self.cfg, self.S, self.M = cfg, max_sessions, n_modules
        # sessions whose prefills share one batched forward (run_batch):
        # 2 x 4k tokens per GEMM is 3% faster than one at a time on B200
        self.prefill_group = max(1, prefill_group)
        self.max_prompt, self.max_new = max_prompt, max_new
        torch.cuda.set_device(device)
        self.base = base or ModuleWeights(cfg, seed, device=device, with_head=False)
        self.mods = modules or [ModuleWeights(cfg, seed + 1 + i, device=device)
                                for i in range(n_modules)]
        self.priv_pages = (max_new + PAGE_TOKENS - 1) // PAGE_TOKENS
        # every session of a full batch holds its whole prompt's full blocks
        # pinned until its decode is done
        if pool_pages < max_sessions * (max_prompt // PAGE_TOKENS):
            raise ValueError(f"pool_pages {pool_pages} < max_sessions x full blocks per prompt "
                             f"({max_sessions * (max_prompt // PAGE_TOKENS)})")
        self.pool_pages = pool_pages
        extra = max_sessions * (1 + n_modules * self.priv_pages)
        self.kv = KVCache(cfg, pool_pages + extra, device)
        # the pool's kernels and host syncs run on their own (high-priority)
        # stream: a lookup for the next sessions does not wait for the
        # prefills already queued, so the host stays ahead of the GPU
        self.pool_stream = torch.cuda.Stream(device=device, priority=-1)
        self.pool = BlockPool(capacity_blocks=pool_pages, block_size=PAGE_TOKENS, device=device,
                              stream=self.pool_stream.cuda_stream,
                              kv_pages=pool_pages, max_query_tokens=max(1 << 17, max_prompt))
        self.prefill = PrefillRunner(cfg, self.base, self.kv, max_tokens=max_prompt * self.prefill_group,
                                     device=device)
        self.tail_page = [pool_pages + s for s in range(max_sessions)]
        nxt = pool_pages + max_sessions
        rows = []
        for s in range(max_sessions):
            for m in range(n_modules):
                rows.append(DecodeRow(module=m, session=s, first_token=0,
                                      pages=list(range(nxt, nxt + self.priv_pages))))
                nxt += self.priv_pages
        max_sp = (max_prompt + PAGE_TOKENS - 1) // PAGE_TOKENS
        sessions = [SessionSpec(shared_len=1, pages=[self.tail_page[s]] * max_sp)
                    for s in range(max_sessions)]
        self.batch = DecodeBatch(sessions, rows, n_modules, device)
        self.runner = DecodeRunner(cfg, self.mods, self.kv, self.batch, max_new, device=device)
        self.dev = torch.device("cuda", device)
        self._tok_dev = torch.empty(max_sessions, max_prompt, dtype=torch.int64, device=self.dev)
        self._tok_host = torch.empty(max_sessions, max_prompt, dtype=torch.int64).pin_memory()
        self._out_host = torch.empty(max_sessions * n_modules, max_new, dtype=torch.int32).pin_memory()
        self._now = 0

    # -- bookkeeping ---------------------------------------------------------

    def launches_per_serve(self, n_sessions: int, prefill_sessions: int, new_tokens: int | None = None) -> int:
        """Kernel launches of ours per serve(): pool (lookup, insert, pin,
        release x2) + prefill (in groups of prefill_group sessions; K3 once
        per sequence when every sequence has >= 1024 new tokens) + decode
        steps."""
        from .model import PER_SEQ_ATTN_MIN_TOKENS
        new_tokens = self.max_prompt if new_tokens is None else new_tokens
        pre, left = 0, prefill_sessions
        while left > 0:
            g = min(left, self.prefill_group)
            attn = g if (g == 1 or new_tokens >= PER_SEQ_ATTN_MIN_TOKENS) else 1
            pre += 1 + (self.cfg.n_layers - 1) * (6 + attn) + 2  # kv_only: the last layer stops after QKV
            left -= g
        return 5 * n_sessions + pre + self.max_new * self.runner.launches_per_step

    def capture(self) -> None:
        self.runner.capture()

    # -- serving ---------------------------------------------------------------

    def serve(self, prompts, now: int | None = None, device_tokens: torch.Tensor | None = None) -> ServeResult:
        """Serve one batch: every session's prompt through the shared prefill,
        then every decode module on every session.

        prompts: list of 1-D int64 arrays (host). With device_tokens (an
        int64 [S, max_prompt] device tensor already holding the prompts) the
        host->device copy is skipped (inputs resident in HBM)."""
        S = len(prompts)
        if S > self.S:
            raise ValueError("more sessions than the engine was built for")
        self._now = self._now + 1 if now is None else now
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        now = self._now
        lens = [len(p) for p in prompts]
        if max(lens) > self.max_prompt or min(lens) < 2:
            raise ValueError("prompt length outside [2, max_prompt]")
        if device_tokens is None:
            for s, p in enumerate(prompts):
                self._tok_host[s, :lens[s]] = torch.from_numpy(np.asarray(p, dtype=np.int64))
            self._tok_dev[:S].copy_(self._tok_host[:S], non_blocking=True)
            toks = self._tok_dev
        else:
            toks = device_tokens
        matched, pref, held, tables, pending = [], [], [], [], []
        try:
            for s, p in enumerate(prompts):
                n = lens[s]
                m, chain = self.pool.longest_prefix_match(SHARED_NS, p, now)
                held.append(chain)  # pinned by the match (kvstore.py:131-134)
                new = self.pool.insert(SHARED_NS, p, now)
                self.pool.pin(new, now)
                held.append(new)
                pages = chain.slots.tolist() + new.slots.tolist()
                if n % PAGE_TOKENS:
                    pages.append(self.tail_page[s])
                if n > m:
                    pending.append((toks[s, m:n], m, pages))
                    if len(pending) == self.prefill_group:
                        self.prefill.run_batch(pending, kv_only=True)
                        pending = []
                matched.append(m)
                pref.append(n - m)
                tables.append(pages)
            if pending:
                self.prefill.run_batch(pending, kv_only=True)
            # decode modules read the base KV of positions [0, n-1) and process the
            # last prompt token themselves (model.ts:372-374, evaluate.ts:16-19)
            while len(tables) < self.S:  # idle session slots: point at a valid page
                tables.append([self.tail_page[len(tables)]])
            lens_full = [n - 1 for n in lens] + [0] * (self.S - S)
            firsts = [int(p[-1]) for p in prompts] + [0] * (self.S - S)
            self.batch.update_sessions(lens_full, tables, firsts)
            ev[1].record()
            out = self.runner.run(self.max_new)
            ev[2].record()
            self._out_host.copy_(out, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        finally:
            # pins drop (cluster.py:404-412) also when an op raised: a failed
            # serve must not leak pinned capacity (cluster.py:348-350)
            torch.cuda.current_stream().synchronize()
            # one release call for the whole batch: the same per-block sequence
            # as releasing the chains one by one (kvstore.py:242-250), one
            # launch + sync instead of 2 per session
            if held:
                slots = np.concatenate([h.slots for h in held])
                ids = np.concatenate([h.ids for h in held])
                for i in range(0, len(ids), self.pool.max_handles):
                    self.pool.release(BlockChain(self.pool, slots[i:i + self.pool.max_handles],
                                                 ids[i:i + self.pool.max_handles]))
        # device time of the two phases (prefill phase includes the pool ops' gaps)
        self.last_phase_ms = {"prefill": ev[0].elapsed_time(ev[1]), "decode": ev[1].elapsed_time(ev[2])}
        res = self._out_host.numpy().reshape(self.S, self.M, self.max_new)[:S].copy()
        return ServeResult(tokens=res, matched=matched, prefill_tokens=pref)
