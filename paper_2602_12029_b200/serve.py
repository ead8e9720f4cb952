"""Real-time multi-model agent serving on one B200 (BASELINE configs 3 / 5).

Drives the reference's agent workload (workload.generate: Poisson sessions,
agent chains rotated per session, synthetic packed token ids) through real
GPU work with the reference's request life cycle (src/prefillsim/cluster.py):

  arrival / admission      cluster.py:256-269 (admission cap)
  dispatch                 cluster.py:271-318 (context = prompt + extensions +
                           outputs; first request issued at session arrival)
  prefill                  cluster.py:322-366: pool lookup (pins) -> forward of
                           the uncached tokens -> insert + pin; in BASELINE mode
                           the request's own model prefills under its own
                           namespace, in PREFILLSHARE mode the frozen base
                           prefills under the shared one (router.py:53-56)
  decode                   cluster.py:414-442: one batched step advances every
                           active request of every model (continuous batching,
                           grouped GEMV over the modules, K6 attention)
  completion               cluster.py:446-478: output appended (synth ids),
                           next agent of the chain dispatched

Decode rows are fixed slots (rows_per_module per model) so one CUDA graph
serves every step; a request takes a free slot of its model. Control flow
needs no device->host sync per step: a request of output_len L finishes after
exactly L steps (the reference appends synthetic output ids, not the
generated ones: cluster.py:453-457).
"""

from __future__ import annotations

import json
import math
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import workload as wl
from .kvstore import BlockPool
from .model import (PAGE_TOKENS, DecodeBatch, DecodeRow, DecodeRunner, KVCache, LlamaConfig,
                    ModuleWeights, PrefillRunner, SessionSpec)
from .router import Router, ServingMode
from .staging import HostKVTier, block_edges, block_keys


@dataclass
class RequestRecord:
    request_id: int
    session_id: int
    model_id: str
    issue_us: float
    first_token_us: float | None = None
    done_us: float | None = None
    out_tokens: int = 0
    matched: int = 0
    prefilled: int = 0
    failed: bool = False


TRACE_KINDS = ("SessionArrival", "PrefillStart", "PrefillComplete", "HandoffComplete", "DecodeStep",
               "RequestComplete", "SessionComplete")  # core.py:124-131


def trace_line(t_us: float, seq: int, kind: str, session: int = -1, request: int = -1, worker: int = -1,
               detail: str = "") -> str:
    """SimEvent.trace_line (core.py:146-150), byte for byte."""
    return f"{int(t_us)} {seq} {kind} {session} {request} {worker} {detail}"


@dataclass
class _Req:
    rec: RequestRecord
    session: int
    ctx: np.ndarray
    output_len: int
    model_idx: int
    worker: int = 0


@dataclass
class _Row:
    req: _Req | None = None
    steps: int = 0
    held: list = field(default_factory=list)
    pool: BlockPool | None = None
    ready: bool = True            # handoff="copy": its context is resident in decode pages
    dpages: list = field(default_factory=list)


class AgentServer:
    def __init__(self, cfg: LlamaConfig, model_ids: list[str], mode: ServingMode, *,
                 rows_per_module: int = 8, pool_pages_per_worker: int = 2048, max_context: int = 4096,
                 max_output: int = 256, seed: int = 0, device: int = 0,
                 modules: list[ModuleWeights] | None = None, base: ModuleWeights | None = None,
                 prefill_batch: bool = True, host_tier_blocks: int = 0, merged_pool: bool = False,
                 handoff: str = "pin", decode_capacity_blocks: int = 4500, staging_threshold: float = 0.9):
        self.cfg, self.mode, self.model_ids = cfg, mode, list(model_ids)
        self.prefill_batch = prefill_batch
        self.trace: list[str] | None = None
        self._trace_raw: list | None = None
        self._fail_reason = ""
        self._pending: list = []
        self._pending_slots: set = set()
        M = len(model_ids)
        self.router = Router(mode, model_ids)
        self.mods = modules or [ModuleWeights(cfg, seed + 1 + i, device=device) for i in range(M)]
        self.base = None
        if mode is ServingMode.PREFILLSHARE:
            self.base = base or ModuleWeights(cfg, seed, device=device, with_head=False)
        # KV pages: [worker pools ...][row tail pages][row private pages]. The
        # reference fleet has one prefill worker (and pool, with its own LRU)
        # per model (cluster.py:156-160). BASELINE routes each request to its
        # model's worker; PREFILLSHARE pins each session to the least-queued
        # worker (router.py:58-77), every worker running the frozen base
        # module. merged_pool=True instead gives PREFILLSHARE ONE shared pool
        # of the same total capacity (one global LRU; a variant, not the
        # reference fleet).
        n_workers = 1 if (mode is ServingMode.PREFILLSHARE and merged_pool) else M
        per_pool = M * pool_pages_per_worker // n_workers
        self.priv_pages = (max_output + PAGE_TOKENS - 1) // PAGE_TOKENS
        self.R = M * rows_per_module
        # handoff="pin": the decode rows read the prefill pool's pages in
        # place (zero copy on one GPU; the pins last until the request
        # completes). handoff="copy": the reference's fleet semantics -- the
        # context moves into its decode worker's own KV budget
        # (decode_capacity_blocks per model, config.py:40) and the prefill
        # pins drop at handoff (cluster.py:404-412); a handoff arriving while
        # the decode worker's resident fraction exceeds staging_threshold
        # (or that does not fit) is staged in pinned host memory and
        # reloaded when the budget has room (costs.py:66-83, App. B)
        if handoff not in ("pin", "copy"):
            raise ValueError("handoff must be 'pin' or 'copy'")
        self.handoff = handoff
        dec_pages = M * decode_capacity_blocks if handoff == "copy" else 0
        total = n_workers * per_pool + self.R * (1 + self.priv_pages) + dec_pages
        self.kv = KVCache(cfg, total, device)
        # each logical prefill worker owns a disjoint page range of the one cache
        self.pools = []
        # pool kernels + their host syncs on a side stream: a lookup does not
        # wait for the prefill forwards and decode steps already queued
        self.pool_stream = torch.cuda.Stream(device=device, priority=-1)
        for w in range(n_workers):
            p = BlockPool(per_pool, PAGE_TOKENS, device=device, kv_pages=per_pool,
                          max_query_tokens=max(1 << 16, max_context), stream=self.pool_stream.cuda_stream)
            p.page_base = w * per_pool
            self.pools.append(p)
        producers = [self.base] if self.base is not None else self.mods
        self.prefillers = [PrefillRunner(cfg, w, self.kv, max_tokens=max_context, device=device)
                           for w in producers]
        rows, sessions = [], []
        nxt = n_workers * per_pool
        self.tail_page = []
        for r in range(self.R):
            self.tail_page.append(nxt)
            nxt += 1
        max_sp = (max_context + PAGE_TOKENS - 1) // PAGE_TOKENS + 1
        for m in range(M):
            for k in range(rows_per_module):
                r = m * rows_per_module + k
                rows.append(DecodeRow(module=m, session=r, first_token=0,
                                      pages=list(range(nxt, nxt + self.priv_pages))))
                nxt += self.priv_pages
                sessions.append(SessionSpec(shared_len=0, pages=[self.tail_page[r]] * max_sp))
        self.batch = DecodeBatch(sessions, rows, M, device)
        self.runner = DecodeRunner(cfg, self.mods, self.kv, self.batch, max_output, device=device)
        self.rows = [_Row() for _ in range(self.R)]
        self.rows_per_module = rows_per_module
        self.residency = []
        self._handoffs: list = []
        self._staged: list[deque] = [deque() for _ in range(M)]
        if handoff == "copy":
            from .staging import DecodeResidency
            first = total - dec_pages
            self.residency = [DecodeResidency(self.kv, first + m * decode_capacity_blocks, decode_capacity_blocks,
                                              staging_threshold) for m in range(M)]
        # host staging tier behind the prefix pool(s) (staging.py; 0 = off)
        self.tier = HostKVTier(self.kv, host_tier_blocks) if host_tier_blocks > 0 else None
        self._pending_store: list = []
        self.max_context, self.max_output = max_context, max_output
        self.dev = torch.device("cuda", device)

    # -- helpers -------------------------------------------------------------

    def _row_of_module(self, m: int) -> int | None:
        for k in range(self.rows_per_module):
            r = m * self.rows_per_module + k
            if self.rows[r].req is None:
                return r
        return None

    def _vocab_ids(self, ctx: np.ndarray) -> torch.Tensor:
        # model inputs: packed synthetic ids folded into the vocabulary
        return torch.from_numpy((ctx % self.cfg.vocab).astype(np.int64)).to(self.dev, non_blocking=True)

    def _prefill(self, req: _Req, now_us: int):
        """cluster.py:322-366 pool side: lookup (pins), insert + pin of the
        new blocks, decode row claimed. The forward itself is queued in
        self._pending and run by _flush_prefills (batched per prefill
        module). Returns (held handles, page table, matched tokens,
        prefilled tokens, decode row), or None on CapacityExhausted."""
        worker = self.router.route_prefill(req.rec, self._queue_depths())
        req.worker = worker
        self._emit(now_us, "PrefillStart", req.session, req.rec.request_id, worker)
        pool = self.pools[worker]
        ns = self.router.prefill_namespace(req.rec.model_id)
        n = len(req.ctx)
        m, chain = pool.longest_prefix_match(ns, req.ctx, now_us)
        base = pool.page_base
        hit = [base + s for s in chain.slots.tolist()]
        if self._pending_slots.intersection(hit):
            # this prefix is written by a forward still queued in the batch
            self._flush_prefills()
        try:
            new = pool.insert(ns, req.ctx, now_us)
        except pool.CapacityError as exc:
            # cluster.py:348-350: release the matched pins and fail the request
            pool.release(chain)
            self._fail_reason = str(exc)
            return None
        pool.pin(new, now_us)
        fresh = [base + s for s in new.slots.tolist()]
        pages = hit + fresh
        row = self._row_of_module(req.model_idx)
        if n % PAGE_TOKENS:
            pages.append(self.tail_page[row])
        # partial prefill from the last cached full block; the tail block is recomputed
        nfull = n // PAGE_TOKENS
        pos0 = min(m, nfull * PAGE_TOKENS)
        if self.tier is not None and nfull > 0:
            # GPU misses found in the host tier are reloaded instead of recomputed
            keys = block_keys(ns, req.ctx, nfull)
            mb = m // PAGE_TOKENS
            slots = self.tier.lookup(keys[mb:nfull], block_edges(ns, req.ctx, keys, mb, nfull))
            if slots:
                self.tier.reload(slots, fresh[:len(slots)])
            pos0 = min(m + PAGE_TOKENS * len(slots), nfull * PAGE_TOKENS)
            h = len(slots)
            if nfull - mb > h:  # write-through of the blocks this forward computes
                self._pending_store.append((keys[mb + h:nfull], block_edges(ns, req.ctx, keys, mb + h, nfull),
                                            fresh[h:nfull - mb]))
        # cluster.py:333-337 / 384-389: the reference's matched / new split;
        # stamped when the forward that computes the request's KV has run on
        # the GPU (immediately when nothing is left to compute)
        done_info = (req.session, req.rec.request_id, worker, m, n, self.handoff == "pin")
        if n > pos0:
            ri = 0 if self.base is not None else req.model_idx
            self._pending.append((ri, self._vocab_ids(req.ctx[pos0:]), pos0, pages, done_info))
            self._pending_slots.update(fresh)
            if not self.prefill_batch:
                self._flush_prefills()
        else:
            self._prefill_done(now_us, done_info)
        return [(pool, chain), (pool, new)], pages, m, n - pos0, row

    def _queue_depths(self) -> list[int]:
        """Per prefill worker: queued forwards + 1 if one is running on the GPU
        (cluster.py:310, len(queue) + busy). A worker's forward is queued
        while it waits in the batch, running until its completion event
        fires."""
        d = [0] * len(self.pools)
        for *_, info in self._pending:
            d[info[2]] += 1
        self._poll()
        busy = {info[2] for item in self._inflight if item[0] == "prefill" for info in item[2]}
        for w in busy:
            d[w] += 1
        return d

    def _prefill_done(self, t_us: float, info) -> None:
        sess, rid, worker, m, n, handoff_too = info
        self._emit(t_us, "PrefillComplete", sess, rid, worker, f"matched={m} new={n - m}")
        if handoff_too:  # handoff="pin": zero copy, complete with the prefill
            self._emit(t_us, "HandoffComplete", sess, rid, worker, f"tokens={n} staged=0")

    # -- handoff="copy": decode-side residency and staging --------------------

    def _hand_off(self) -> None:
        """Move the contexts whose prefill forwards are queued into their
        decode workers' budgets (K8 page copy, ordered after the forward) or
        stage them to host memory; drop the prefill pins (cluster.py:404-412)."""
        for req, row, pages, held, worker in self._handoffs:
            res = self.residency[req.model_idx]
            n = len(pages)
            if n > res.capacity:
                raise ValueError(f"a {n}-page context exceeds the decode budget of {res.capacity} pages "
                                 "(decode_capacity_blocks)")
            if res.must_stage(n):
                self._staged[req.model_idx].append((req, row, res.stage(pages), n, worker))
            else:
                dp = res.take(n)
                from .transfer import copy_pages
                copy_pages(self.kv.data.view(self.kv.n_pages, -1), self.kv.data.view(self.kv.n_pages, -1), pages, dp)
                self._activate(req, row, dp, worker, staged=False)
            for pool, h in held:
                pool.release(h)
            self.rows[row].held = []
        self._handoffs = []

    def _reload_staged(self) -> None:
        """Staged contexts back into decode pages, FIFO per decode worker,
        as its budget frees up."""
        for m, q in enumerate(self._staged):
            res = self.residency[m] if self.residency else None
            while q and res.can_take(q[0][3]):
                req, row, host, n, worker = q.popleft()
                dp = res.take(n)
                res.reload(host, dp)
                self._activate(req, row, dp, worker, staged=True)

    def _activate(self, req, row, dpages, worker, staged: bool) -> None:
        r = self.rows[row]
        r.dpages, r.ready = dpages, True
        self.batch.update_row(row, len(req.ctx) - 1, dpages, int(req.ctx[-1] % self.cfg.vocab))
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self._inflight.append(("handoff", ev, [(req.session, req.rec.request_id, worker, len(req.ctx), staged)]))

    def _flush_prefills(self) -> None:
        """Run the queued forwards: one batched forward per prefill module and
        <= max_context stacked tokens (small partial
        prefills share each layer's weight stream)."""
        by_runner: dict[int, list] = {}
        for ri, toks, pos0, pages, info in self._pending:
            by_runner.setdefault(ri, []).append((toks, pos0, pages, info))
        self._pending, self._pending_slots = [], set()
        if self.tier is not None:
            self.tier.fence()
        for res in self.residency:  # pending stagings read pages these forwards may overwrite
            res.fence()
        for ri, seqs in by_runner.items():
            runner = self.prefillers[ri]
            chunk, tot = [], 0
            for sq in seqs + [None]:
                if sq is None or (chunk and tot + int(sq[0].shape[0]) > runner.max_tokens):
                    ev = self._events("prefill")
                    runner.run_batch([c[:3] for c in chunk], kv_only=True)  # decode processes the last token
                    ev[1].record()
                    self._inflight.append(("prefill", ev[1], [c[3] for c in chunk]))
                    chunk, tot = [], 0
                if sq is not None:
                    chunk.append(sq)
                    tot += int(sq[0].shape[0])
        if self.tier is not None:
            for keys, edges, pages in self._pending_store:
                self.tier.store(keys, edges, pages)
            self._pending_store = []

    def _emit(self, t_us: float, kind: str, session: int = -1, request: int = -1, worker: int = -1,
              detail: str = "") -> None:
        """One trace event in the reference's format (core.py:146-150):
        `time seq kind session request worker detail`; time = us since the
        run started: host time for arrivals / prefill starts, the GPU
        completion time (CUDA events) for prefill, handoff, decode steps and
        completions. Lines are ordered by time (seq follows) when the run
        ends."""
        if self._trace_raw is not None:
            self._trace_raw.append((t_us, kind, session, request, worker, detail))

    def _dev_us(self, ev) -> float:
        """GPU completion time of a recorded event, in us since the run started."""
        return self._clk0.elapsed_time(ev) * 1e3

    def _poll(self) -> None:
        """Stamp every completed prefill forward / decode step (in stream
        order) with its GPU completion time: PrefillComplete / HandoffComplete
        trace lines, first-token times (TTFT includes the request's own
        prefill and its first decode step), token completions."""
        while self._inflight and self._inflight[0][1].query():
            item = self._inflight.popleft()
            t = self._dev_us(item[1])
            if item[0] == "prefill":
                for info in item[2]:
                    self._prefill_done(t, info)
            elif item[0] == "handoff":
                for sess, rid, worker, n, staged in item[2]:
                    self._emit(t, "HandoffComplete", sess, rid, worker, f"tokens={n} staged={int(staged)}")
            else:
                _, _, first, n_busy, per_model = item
                for rec in first:
                    rec.first_token_us = t
                self.token_completions.append((int(t), n_busy))  # cluster.py:434
                M = len(self.model_ids)
                for m, nb in enumerate(per_model):  # one DecodeStep per decode worker with rows in flight
                    if nb:
                        self._emit(t, "DecodeStep", worker=M + m, detail=f"batch={nb}")

    def _events(self, kind: str):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        self._ev.append((kind, a, b))
        return a, b

    def gpu_time(self) -> dict:
        """Device time spent in prefill forwards and decode steps over the
        last run() (CUDA events around each launch sequence)."""
        out = {"prefill_ms": 0.0, "decode_ms": 0.0, "prefill_calls": 0, "decode_steps": 0}
        for kind, a, b in self._ev:
            out[kind + "_ms"] += a.elapsed_time(b)
            out["prefill_calls" if kind == "prefill" else "decode_steps"] += 1
        return {k: round(v, 1) if isinstance(v, float) else v for k, v in out.items()}

    # -- serving -------------------------------------------------------------

    def run(self, sessions: list[wl.SessionSpec], max_concurrent: int | None = None,
            time_scale: float = 1.0, record_trace: bool = False) -> list[RequestRecord]:
        """Serve the workload in real time (arrival times scaled by
        time_scale). Returns one record per request. record_trace: keep the
        event trace (self.trace, the reference's trace.txt lines)."""
        self.trace = None
        self._trace_raw = [] if record_trace else None
        self.runner.capture()
        self._ev = []
        self._inflight: deque = deque()
        self.token_completions: list[tuple[int, int]] = []
        st = torch.cuda.current_stream()
        st.synchronize()
        self._clk0 = torch.cuda.Event(enable_timing=True)
        records: list[RequestRecord] = []
        arrivals = deque(sorted(sessions, key=lambda s: s.arrival_time))
        waiting_admission: deque = deque()
        active = 0
        cap = max_concurrent or (1 << 30)
        ctx: dict[int, list] = {}
        step_idx: dict[int, int] = {}
        spec_of = {s.session_id: s for s in sessions}
        prefill_q: deque[_Req] = deque()
        next_rid = [0]
        t0 = time.perf_counter()
        self._clk0.record(st)  # the GPU clock's origin (the stream is idle)

        def now_us() -> float:
            return (time.perf_counter() - t0) * 1e6

        def dispatch(sid: int, issue_us: float):
            spec = spec_of[sid]
            k = step_idx[sid]
            agent = spec.agent_chain[k % len(spec.agent_chain)]
            ctx[sid].extend(wl.synth_tokens(sid, wl.extension_slot(k), agent.input_extension_len))
            rec = RequestRecord(next_rid[0], sid, agent.model_id, issue_us)
            next_rid[0] += 1
            records.append(rec)
            prefill_q.append(_Req(rec, sid, np.array(ctx[sid], dtype=np.int64), agent.output_len,
                                  self.model_ids.index(agent.model_id)))

        def activate(spec):
            ctx[spec.session_id] = list(wl.synth_tokens(spec.session_id, wl.prompt_slot(),
                                                       spec.initial_prompt_len))
            step_idx[spec.session_id] = 0
            dispatch(spec.session_id, spec.arrival_time * time_scale)  # counts admission wait

        done_sessions = 0
        n_sessions = len(sessions)
        while done_sessions < n_sessions:
            t = now_us()
            while arrivals and arrivals[0].arrival_time * time_scale <= t:
                s = arrivals.popleft()
                self._emit(t, "SessionArrival", s.session_id)
                if active < cap:
                    active += 1
                    activate(s)
                else:
                    waiting_admission.append(s)
            # prefills whose model has a free decode row (handoff = zero-copy pin)
            progressed = False
            for _ in range(len(prefill_q)):
                req = prefill_q.popleft()
                if self._row_of_module(req.model_idx) is None:
                    prefill_q.append(req)
                    continue
                got = self._prefill(req, int(now_us()))
                progressed = True
                if got is None:
                    # cluster.py:480-490: the request and its session fail
                    req.rec.failed = True
                    self._emit(now_us(), "SessionComplete", req.session, detail=f"failed: {self._fail_reason}")
                    done_sessions += 1
                    active -= 1
                    if waiting_admission:
                        active += 1
                        activate(waiting_admission.popleft())
                    continue
                held, pages, m, pre, row = got
                req.rec.matched, req.rec.prefilled = m, pre
                r = self.rows[row]
                r.req, r.steps, r.held = req, 0, held
                if self.handoff == "copy":  # moved into decode pages after its forward is queued
                    r.ready = False
                    self._handoffs.append((req, row, pages, held, req.worker))
                else:
                    self.batch.update_row(row, len(req.ctx) - 1, pages, int(req.ctx[-1] % self.cfg.vocab))
                progressed = True
            if self._pending:
                self._flush_prefills()
            if self._handoffs:
                self._hand_off()
            if self.handoff == "copy":
                self._reload_staged()
            self._poll()
            busy = [r for r in self.rows if r.req is not None and r.ready]
            if busy:
                ev = self._events("decode")
                self.runner.graph.replay()
                ev[1].record()
                per_model = [0] * len(self.model_ids)
                for r in busy:
                    per_model[r.req.model_idx] += 1
                first = [r.req.rec for r in busy if r.steps == 0]
                self._inflight.append(("step", ev[1], first, len(busy), per_model))
                for idx, r in enumerate(self.rows):
                    if r.req is None or not r.ready:
                        continue
                    r.steps += 1
                    rec = r.req.rec
                    if r.steps >= r.req.output_len:
                        ev[1].synchronize()
                        self._poll()
                        rec.done_us = self._dev_us(ev[1])
                        rec.out_tokens = r.steps
                        self._emit(rec.done_us, "RequestComplete", r.req.session, rec.request_id,
                                   len(self.model_ids) + r.req.model_idx)
                        for pool, h in r.held:
                            pool.release(h)
                        if r.dpages:  # handoff="copy": the context leaves the decode budget
                            self.residency[r.req.model_idx].give(r.dpages)
                        sid = r.req.session
                        spec = spec_of[sid]
                        ctx[sid].extend(wl.synth_tokens(sid, wl.output_slot(step_idx[sid]), r.req.output_len))
                        step_idx[sid] += 1
                        self.rows[idx] = _Row()
                        self.batch.update_row(idx, 0, [self.tail_page[idx]], 0)
                        if step_idx[sid] >= spec.total_requests:
                            self._emit(rec.done_us, "SessionComplete", sid)
                            done_sessions += 1
                            active -= 1
                            if waiting_admission:
                                active += 1
                                activate(waiting_admission.popleft())
                        else:
                            dispatch(sid, rec.done_us)
            elif not progressed:
                if any(self._staged):
                    continue  # staged contexts wait for a decode budget that only completions free
                if arrivals:
                    wait = arrivals[0].arrival_time * time_scale - now_us()
                    if wait > 0:
                        time.sleep(min(wait / 1e6, 0.05))
                elif not prefill_q:
                    break
        st.synchronize()
        self._poll()
        if self._trace_raw is not None:  # (time, seq) order; stable for equal times
            self.trace = [trace_line(e[0], i, *e[1:])
                          for i, e in enumerate(sorted(self._trace_raw, key=lambda e: e[0]))]
        return records


def summarize(records: list[RequestRecord], warmup_fraction: float = 0.1) -> dict:
    """metrics.py:22-76 definitions (nearest-rank p95, post-warmup window),
    plus req/s over the same window."""
    done = [r for r in records if r.done_us is not None]
    failed = sum(1 for r in records if r.failed)
    if not done:
        return {"completed": 0, "failed": failed}
    t_end = max(r.done_us for r in done)
    w0 = warmup_fraction * t_end
    win = [r for r in done if r.done_us >= w0]
    window_s = (t_end - w0) / 1e6
    e2e = sorted(r.done_us - r.issue_us for r in done)
    ttft = sorted(r.first_token_us - r.issue_us for r in done if r.first_token_us is not None)

    def p95(v):
        return v[max(math.ceil(0.95 * len(v)), 1) - 1]

    lookup = sum(r.matched + r.prefilled for r in done)
    return {"completed": len(done), "failed": failed, "req_per_s": len(win) / window_s,
            "tok_per_s": sum(r.out_tokens for r in win) / window_s,
            "p95_e2e_ms": p95(e2e) / 1e3, "p95_ttft_ms": p95(ttft) / 1e3 if ttft else None,
            "prefill_tokens": sum(r.prefilled for r in done),
            "prefix_hit_ratio": sum(r.matched for r in done) / max(1, lookup),
            "wall_s": t_end / 1e6}


# -- the reference's output formats (src/prefillsim/metrics.py:17-91) --------

SCHEMA_VERSION = 1
CSV_HEADER = "request_id,session_id,model_id,ttft_us,e2e_us,out_tokens"


def _percentile(values, p):
    ordered = sorted(values)
    return ordered[max(math.ceil(p / 100.0 * len(ordered)), 1) - 1]


def build_report(server: "AgentServer", records: list[RequestRecord], config_echo: dict,
                 warmup_fraction: float = 0.1) -> dict:
    """report.json of a real-engine run in the reference's versioned schema
    (metrics.py:44-80; pool aggregates as cluster.py:232-252): every field is
    the reference's, measured on the GPU in real time (microseconds since the
    run started) instead of virtual time. staging_handoff_count: handoffs
    staged through host memory (handoff="copy"; 0 with the zero-copy pin
    handoff)."""
    end = max([t for t, _ in server.token_completions] + [int(r.done_us or 0) for r in records] + [0])
    done = [r for r in records if r.done_us is not None and not r.failed]
    ttfts = [int(r.first_token_us - r.issue_us) for r in done if r.first_token_us is not None]
    e2es = [int(r.done_us - r.issue_us) for r in done]
    w0 = warmup_fraction * end
    toks = sum(n for t, n in server.token_completions if t >= w0)
    win = (end - w0) / 1e6
    matched = sum(p.matched_tokens for p in server.pools)
    lookups = sum(p.lookup_tokens for p in server.pools)
    peak: dict[str, int] = {}
    for p in server.pools:
        for ns, t in p.peak_footprint_tokens().items():
            peak[ns] = peak.get(ns, 0) + t
    return {
        "schema_version": SCHEMA_VERSION,
        "config": config_echo,
        "metadata": {
            "hit_ratio_definition": "cumulative matched_tokens / lookup_tokens over prefill lookups",
            "throughput_definition": "generated output tokens completed in the post-warmup window",
            "warmup_fraction": warmup_fraction,
            "engine": "paper_2602_12029_b200 on one B200 (real time)",
        },
        "end_time_us": end,
        "request_count": len(records),
        "completed_count": len(done),
        "failure_count": sum(1 for r in records if r.failed),
        "staging_handoff_count": sum(r.staged_count for r in getattr(server, "residency", [])),
        "p95_e2e_us": _percentile(e2es, 95) if e2es else None,
        "mean_ttft_us": sum(ttfts) / len(ttfts) if ttfts else None,
        "p95_ttft_us": _percentile(ttfts, 95) if ttfts else None,
        "throughput_tok_per_s": toks / win if win > 0 else 0.0,
        "prefix_hit_ratio": matched / lookups if lookups else 0.0,
        "matched_tokens": matched,
        "lookup_tokens": lookups,
        "eviction_count": sum(p.eviction_count for p in server.pools),
        "peak_footprint_tokens": dict(sorted(peak.items())),
        "peak_footprint_total": sum(peak.values()),
    }


def report_to_json(report: dict) -> str:
    return json.dumps(report, sort_keys=True, indent=1)


def records_to_csv(records: list[RequestRecord]) -> str:
    """requests.csv (metrics.py:86-94), one line per request in issue order."""
    lines = [CSV_HEADER]
    for r in sorted(records, key=lambda x: x.request_id):
        ttft = "" if r.first_token_us is None or r.failed else str(int(r.first_token_us - r.issue_us))
        e2e = "" if r.done_us is None or r.failed else str(int(r.done_us - r.issue_us))
        lines.append(f"{r.request_id},{r.session_id},{r.model_id},{ttft},{e2e},{r.out_tokens}")
    return "\n".join(lines) + "\n"
