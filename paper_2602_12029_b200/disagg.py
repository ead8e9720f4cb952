"""Prefill / decode disaggregation across processes (BASELINE
configs 3 and 5): P logical prefill workers and one decode worker per model,
placed on ranks (one process per GPU) by router.Placement.

The request life cycle is the reference fleet's (src/prefillsim/cluster.py):

  dispatch      coordinator (rank 0): session arrivals, agent chain, context
                = prompt + extensions + outputs (cluster.py:256-318)
  prefill       the routed prefill worker: pool lookup (pins) -> forward of
                the uncached tokens -> insert + pin (cluster.py:322-366)
  handoff       the FULL context's KV pages move to the model's decode worker
                (cluster.py:370-412); prefill pins drop afterwards, the
                blocks stay cached for future prefix hits
  decode        continuous batching on the decode worker (cluster.py:414-442)
  completion    output appended, the session's next request dispatched
                (cluster.py:446-478)

Rounds. Every rank runs the same loop. Rank 0 plans a round (the prefills
to run, per prefill worker, and how many decode steps), broadcasts it on a
gloo control group, and every rank executes its part:

  1. prefill workers on this rank: pool ops + ONE batched forward per
     worker (PrefillRunner.run_batch);
  2. handoff: every page of every context moves prefill rank -> decode rank
     in one batch_isend_irecv per rank (NCCL over NVLink on GPUs, gloo on
     CPU; page counts are known from the context lengths, so no headers and
     no send/recv ordering deadlock); a handoff inside one rank is a page
     copy (K8 on GPUs);
  3. decode workers: admit the received contexts into free rows, run the
     round's decode steps;
  4. reports (prefill hits, completions) gather to rank 0.

Prefill of round r+1 overlaps decode of round r only across GPUs (different
ranks), which is what disaggregation buys. The compute is behind two small
backend interfaces so the protocol runs on CPU (tests: gloo, world_size 3,
synthetic backends that check every moved page) and on B200s
(GpuPrefillBackend / GpuDecodeBackend: K1-K3, K5-K6, K7, K8).
"""

from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import workload as wl
from .router import Placement, Router, ServingMode

PAGE_TOKENS = 16


# ----------------------------------------------------------------- plans ----

@dataclass
class Job:
    """One request's prefill + handoff, as planned by the coordinator."""
    rid: int
    sid: int
    model: int                 # model index (decode worker)
    ctx: np.ndarray            # full context token ids (int64)
    out_len: int
    worker: int                # logical prefill worker
    src: int = 0               # prefill rank
    dst: int = 0               # decode rank

    @property
    def n_pages(self) -> int:
        return (len(self.ctx) + PAGE_TOKENS - 1) // PAGE_TOKENS


@dataclass
class Round:
    jobs: list[Job]
    steps: int                 # decode steps every decode worker runs this round
    now_us: int
    stop: bool = False


@dataclass
class Record:
    rid: int
    sid: int
    model_id: str
    issue_us: float
    first_token_us: float | None = None
    done_us: float | None = None
    matched: int = 0
    prefilled: int = 0
    out_tokens: int = 0
    failed: bool = False


# -------------------------------------------------------------- backends ----

class PrefillBackend:
    """What a prefill worker needs: the reference BlockPool API (`pool`), the
    KV page store (`kv_pages`: [n_pages, page_elems] tensor, the unit of the
    handoff), the pages the pool's slots map to, a tail page per in-flight
    request, and the forward of stacked partial prefills."""

    pool = None
    kv_pages: torch.Tensor

    def slot_page(self, slot: int) -> int:
        raise NotImplementedError

    def tail_page(self, k: int) -> int:
        """Scratch page for the partial last block of the k-th job of a round."""
        raise NotImplementedError

    def forward(self, seqs: list[tuple[np.ndarray, int, list[int]]]) -> None:
        """seqs: (token ids of positions [pos0, pos0 + T), pos0, page table)."""
        raise NotImplementedError

    def pack(self, pages: list[int]) -> torch.Tensor:
        """The pages, gathered into one contiguous [n, page] buffer (one P2P
        message per peer per round instead of one per 2 MiB page)."""
        return self.kv_pages[torch.as_tensor(pages, dtype=torch.long, device=self.kv_pages.device)]


class DecodeBackend:
    """What a decode worker needs: a page store with an allocator, a fixed
    number of rows per hosted model, admit / step / retire."""

    kv_pages: torch.Tensor

    def alloc(self, n: int) -> list[int]:
        raise NotImplementedError

    def free(self, pages: list[int]) -> None:
        raise NotImplementedError

    def free_row(self, model: int) -> int | None:
        raise NotImplementedError

    def admit(self, row: int, job: Job, pages: list[int]) -> None:
        raise NotImplementedError

    def retire(self, row: int) -> None:
        raise NotImplementedError

    def step(self) -> None:
        """One decode step of every row (idle rows compute garbage, unread)."""
        raise NotImplementedError

    def mark(self):
        """A completion marker for the step just issued (host backends step
        synchronously: the time is now)."""
        return time.perf_counter()

    def resolve(self, marks: list) -> list[float]:
        """Host perf_counter() times at which the marked steps completed
        (perf_counter is CLOCK_MONOTONIC: one clock for every rank of a node)."""
        return list(marks)

    def copy_pages(self, src: torch.Tensor, src_pages: list[int], dst_pages: list[int]) -> None:
        """Same-rank handoff."""
        for s, d in zip(src_pages, dst_pages):
            self.kv_pages[d].copy_(src[s])

    def unpack(self, buf: torch.Tensor, pages: list[int]) -> None:
        """Scatter a received contiguous buffer into the allocated pages."""
        self.kv_pages[torch.as_tensor(pages, dtype=torch.long, device=self.kv_pages.device)] = buf


# ----------------------------------------------------------- coordinator ----

class Coordinator:
    """Rank 0: the reference's dispatch / completion logic in real time."""

    def __init__(self, sessions: list[wl.SessionSpec], model_ids: list[str], router: Router,
                 placement: Placement, time_scale: float = 1.0, steps_per_round: int = 8):
        self.model_ids = list(model_ids)
        self.router, self.place = router, placement
        self.arrivals = deque(sorted(sessions, key=lambda s: s.arrival_time))
        self.spec = {s.session_id: s for s in sessions}
        self.ctx: dict[int, list] = {}
        self.step_idx: dict[int, int] = {}
        self.queue: deque[Job] = deque()
        self.records: dict[int, Record] = {}
        self.inflight: dict[int, Job] = {}
        self.remaining: dict[int, int] = {}
        self.depth = [0] * len(placement.prefill_gpus)
        self.next_rid = 0
        self.done_sessions = 0
        self.n_sessions = len(sessions)
        self.time_scale = time_scale
        self.steps_per_round = steps_per_round
        self.t0 = time.perf_counter()

    def now_us(self) -> float:
        return (time.perf_counter() - self.t0) * 1e6

    def _dispatch(self, sid: int, issue_us: float) -> None:
        spec = self.spec[sid]
        k = self.step_idx[sid]
        agent = spec.agent_chain[k % len(spec.agent_chain)]
        self.ctx[sid].extend(wl.synth_tokens(sid, wl.extension_slot(k), agent.input_extension_len))
        rid = self.next_rid
        self.next_rid += 1
        self.records[rid] = Record(rid, sid, agent.model_id, issue_us)
        m = self.model_ids.index(agent.model_id)

        class _R:  # what Router.route_prefill reads (router.py:58-77)
            session_id = sid
            model_id = agent.model_id
        w = self.router.route_prefill(_R, self.depth)
        self.depth[w] += 1
        self.queue.append(Job(rid, sid, m, np.asarray(self.ctx[sid], dtype=np.int64), agent.output_len, w,
                              self.place.prefill_gpus[w], self.place.decode_gpus[m]))

    def plan(self, free_rows: dict[tuple[int, int], int]) -> Round:
        """Arrivals up to now, then the queued jobs whose model has a free
        decode row on one of its replicas (free_rows: (model, rank) -> free
        rows after the last round). A job goes to the replica with the most
        free rows (ties -> lowest rank): a placement choice only, the
        logical decode worker (router.py:79-85) is the model's."""
        t = self.now_us()
        while self.arrivals and self.arrivals[0].arrival_time * self.time_scale <= t:
            s = self.arrivals.popleft()
            self.ctx[s.session_id] = list(wl.synth_tokens(s.session_id, wl.prompt_slot(), s.initial_prompt_len))
            self.step_idx[s.session_id] = 0
            self._dispatch(s.session_id, s.arrival_time * self.time_scale)
        jobs, keep = [], deque()
        rows = dict(free_rows)
        while self.queue:
            j = self.queue.popleft()
            best = max(self.place.replicas(j.model), key=lambda g: (rows.get((j.model, g), 0), -g))
            if rows.get((j.model, best), 0) > 0:
                rows[(j.model, best)] -= 1
                j.dst = best
                jobs.append(j)
                self.inflight[j.rid] = j
                self.remaining[j.rid] = j.out_len
            else:
                keep.append(j)
        self.queue = keep
        stop = self.done_sessions >= self.n_sessions
        busy = bool(self.remaining) or bool(jobs)
        if not busy and not stop and self.arrivals:
            wait = self.arrivals[0].arrival_time * self.time_scale - self.now_us()
            if wait > 0:
                time.sleep(min(wait / 1e6, 0.05))
        return Round(jobs, self.steps_per_round if busy else 0, int(t), stop)

    def absorb(self, rnd: Round, prefill_reports: list, decode_reports: list) -> None:
        t = self.now_us()
        for rep in prefill_reports:
            for rid, m, pre, ok in rep:
                rec = self.records[rid]
                rec.matched, rec.prefilled = m, pre
                self.depth[self.inflight[rid].worker] -= 1
                if not ok:  # cluster.py:348-350, 480-490: the request and its session fail
                    rec.failed = True
                    del self.inflight[rid]
                    del self.remaining[rid]
                    self.done_sessions += 1
        for rep in decode_reports:
            for rid, first, n_done, t_abs in rep:
                rec = self.records[rid]
                te = (t_abs - self.t0) * 1e6  # the step's completion on the decode rank
                if first and rec.first_token_us is None:
                    rec.first_token_us = te
                if n_done:
                    rec.done_us = te
                    rec.out_tokens = n_done
                    j = self.inflight.pop(rid)
                    del self.remaining[rid]
                    sid = j.sid
                    self.ctx[sid].extend(wl.synth_tokens(sid, wl.output_slot(self.step_idx[sid]), j.out_len))
                    self.step_idx[sid] += 1
                    if self.step_idx[sid] >= self.spec[sid].total_requests:
                        self.done_sessions += 1
                    else:
                        self._dispatch(sid, max(te, 0.0))


# ----------------------------------------------------------------- ranks ----

class DisaggServer:
    """SPMD serving loop; construct on every rank with the backends this rank
    hosts (prefill: logical worker -> PrefillBackend; decode: the rank's
    DecodeBackend or None)."""

    def __init__(self, placement: Placement, model_ids: list[str], mode: ServingMode,
                 prefill: dict[int, PrefillBackend], decode: DecodeBackend | None,
                 rows_per_model: int, ctrl_group=None, data_group=None):
        self.place, self.model_ids, self.mode = placement, list(model_ids), mode
        self.router = Router(mode, model_ids)
        self.prefill, self.decode = prefill, decode
        self.rows_per_model = rows_per_model
        self.ctrl, self.data = ctrl_group, data_group
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        # decode-side state of this rank: row -> [job, pages, steps done]
        self.rows: dict[int, list] = {}
        # cross-rank handoffs sent by this rank: bytes and sender-side time
        # (pack + transfer, CUDA events on the handoff stream on GPUs)
        self.handoff_bytes = 0
        self.handoff_s = 0.0
        self._hev: list = []
        self._side = None

    # -- one round on this rank ------------------------------------------
    def _prefill_phase(self, rnd: Round):
        """Pool ops + one batched forward per local prefill worker. Returns
        (report, outgoing handoffs [(job, pages)], held pins)."""
        report, out, held = [], [], []
        by_worker: dict[int, list] = {}
        for j in rnd.jobs:
            if j.src == self.rank:
                by_worker.setdefault(j.worker, []).append(j)
        for w, jobs in by_worker.items():
            be = self.prefill[w]
            ns = self.router.prefill_namespace(self.model_ids[jobs[0].model])
            seqs = []
            for k, j in enumerate(jobs):
                ns = self.router.prefill_namespace(self.model_ids[j.model])
                n = len(j.ctx)
                m, chain = be.pool.longest_prefix_match(ns, tuple(int(x) for x in j.ctx), rnd.now_us)
                try:
                    new = be.pool.insert(ns, tuple(int(x) for x in j.ctx), rnd.now_us)
                except be.pool.CapacityError:
                    be.pool.release(chain)
                    report.append((j.rid, m, 0, False))
                    continue
                be.pool.pin(new, rnd.now_us)
                held.append((be.pool, chain))
                held.append((be.pool, new))
                pages = [be.slot_page(s) for s in _slots(chain)] + [be.slot_page(s) for s in _slots(new)]
                if n % PAGE_TOKENS:
                    pages.append(be.tail_page(k))
                pos0 = min(m, (n // PAGE_TOKENS) * PAGE_TOKENS)
                if n > pos0:
                    seqs.append((j.ctx[pos0:], pos0, pages))
                report.append((j.rid, m, n - pos0, True))
                out.append((j, be, pages))
            if seqs:
                be.forward(seqs)
        return report, out, held

    def _stream_ctx(self, t: torch.Tensor):
        """Handoff work on a side stream (GPU): it waits only for the work it
        needs, not for the decode steps queued on the main stream."""
        import contextlib
        if not t.is_cuda:
            return contextlib.nullcontext()
        if self._side is None:
            self._side = torch.cuda.Stream(device=t.device)
        return torch.cuda.stream(self._side)

    def _handoff(self, rnd: Round, out) -> list:
        """All pages of all contexts this round: per (src, dst) rank pair ONE
        contiguous message, the pair's jobs' pages packed in plan order (K8
        page copies on GPUs), exchanged in one batch_isend_irecv per rank
        (NCCL over NVLink on GPUs, gloo on CPU; sizes follow from the context
        lengths, so no headers and no ordering deadlock), unpacked into pages
        from the receiver's allocator. Sender and receiver run it on a side
        stream: the prefill forward it needs is awaited, the receiver's
        queued decode steps are not (the reference serializes ingest with
        decode steps, cluster.py:370-390; here they overlap). A handoff
        inside one rank is a page copy."""
        mine = {j.rid: (be, pages) for j, be, pages in out}
        send: dict[int, list] = {}
        recv: dict[int, list] = {}
        local = []
        for j in rnd.jobs:
            if j.rid not in self._ok_all:
                continue
            if j.src == self.rank and j.dst == self.rank:
                be, pages = mine[j.rid]
                local.append((j, be, pages))
            elif j.src == self.rank:
                send.setdefault(j.dst, []).append(mine[j.rid])
            elif j.dst == self.rank:
                recv.setdefault(j.src, []).append((j, self.decode.alloc(j.n_pages)))
        arrived = []
        if send or recv:
            ref = next(iter(self.prefill.values())).kv_pages if self.prefill else self.decode.kv_pages
            cuda = ref.is_cuda
            main = torch.cuda.current_stream(ref.device) if cuda else None
            with self._stream_ctx(ref):
                if cuda:
                    if send:
                        self._side.wait_stream(main)  # the prefill forwards whose pages are packed
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev0.record()
                t0 = time.perf_counter()
                ops, bufs = [], []
                nbytes = 0
                for dst in sorted(send):
                    parts = [be.pack(pages) for be, pages in send[dst]]
                    buf = parts[0] if len(parts) == 1 else torch.cat(parts)
                    nbytes += buf.numel() * buf.element_size()
                    ops.append(dist.P2POp(dist.isend, buf, dst, group=self.data))
                    bufs.append(buf)
                for src in sorted(recv):
                    n = sum(j.n_pages for j, _ in recv[src])
                    buf = torch.empty((n,) + tuple(self.decode.kv_pages.shape[1:]), dtype=self.decode.kv_pages.dtype,
                                      device=self.decode.kv_pages.device)
                    ops.append(dist.P2POp(dist.irecv, buf, src, group=self.data))
                    bufs.append((src, buf))
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
                if cuda and recv:
                    # freed pages being written may still be read by decode
                    # steps queued before them; the receive itself did not wait
                    self._side.wait_stream(main)
                for item in bufs:
                    if isinstance(item, tuple):
                        src, buf = item
                        off = 0
                        for j, pages in recv[src]:
                            self.decode.unpack(buf[off:off + j.n_pages], pages)
                            off += j.n_pages
                            arrived.append((j, pages))
                if nbytes:
                    self.handoff_bytes += nbytes
                    if cuda:
                        ev1 = torch.cuda.Event(enable_timing=True)
                        ev1.record()
                        self._hev.append((ev0, ev1))
                    else:
                        self.handoff_s += time.perf_counter() - t0
            if cuda:
                main.wait_stream(self._side)  # decode steps read the received pages
        for j, be, pages in local:
            dst = self.decode.alloc(j.n_pages)
            self.decode.copy_pages(be.kv_pages, pages, dst)
            arrived.append((j, dst))
        return arrived

    def handoff_stats(self) -> dict:
        """Bytes this rank sent to other ranks and the sender-side time
        (pack + transfer), GB/s."""
        for a, b in self._hev:
            b.synchronize()
            self.handoff_s += a.elapsed_time(b) / 1e3
        self._hev = []
        return {"bytes": self.handoff_bytes, "seconds": self.handoff_s,
                "gbs": self.handoff_bytes / self.handoff_s / 1e9 if self.handoff_s > 0 else None}

    def _decode_phase(self, rnd: Round, arrived) -> list:
        report = []
        for j, pages in arrived:
            row = self.decode.free_row(j.model)
            assert row is not None, "coordinator over-committed a decode worker"
            self.decode.admit(row, j, pages)
            self.rows[row] = [j, pages, 0]
        marks, pend = [], []
        for _ in range(rnd.steps):
            if not self.rows:
                break
            self.decode.step()
            marks.append(self.decode.mark())
            for row in list(self.rows):
                st = self.rows[row]
                st[2] += 1
                if st[2] == 1:
                    pend.append((st[0].rid, True, 0, len(marks) - 1))
                if st[2] >= st[0].out_len:
                    pend.append((st[0].rid, False, st[2], len(marks) - 1))
                    self.decode.retire(row)
                    self.decode.free(st[1])
                    del self.rows[row]
        # first-token / completion times = when those steps finished on the
        # device (not when they were enqueued)
        times = self.decode.resolve(marks) if marks else []
        for rid, first, n_done, k in pend:
            report.append((rid, first, n_done, times[k]))
        return report

    def free_rows(self) -> dict[tuple[int, int], int]:
        """Free decode rows per (model, this rank) for the replicas hosted here."""
        if self.decode is None:
            return {}
        out = {}
        for m in self.place.decode_models_on(self.rank):
            busy = sum(1 for st in self.rows.values() if st[0].model == m)
            out[(m, self.rank)] = self.rows_per_model - busy
        return out

    def run(self, coord: Coordinator | None, max_rounds: int = 1 << 30) -> dict[int, Record] | None:
        """Serve until every session is done (rank 0 returns the records)."""
        free = self._gather(self.free_rows())
        for _ in range(max_rounds):
            if self.rank == 0:
                rows = {}
                for d in free:
                    rows.update(d)
                rnd = coord.plan(rows)
            else:
                rnd = None
            rnd = self._bcast(rnd)
            if rnd.stop:
                break
            pre_rep, out, held = self._prefill_phase(rnd)
            # every rank needs to know which jobs failed at prefill (no handoff)
            all_pre = self._allgather(pre_rep)
            self._ok_all = {rid for rep in all_pre for rid, _, _, good in rep if good}
            arrived = self._handoff(rnd, out)
            for pool, h in held:  # cluster.py:404-412: pins drop once the handoff is done
                pool.release(h)
            dec_rep = self._decode_phase(rnd, arrived) if self.decode is not None else []
            both = self._gather((dec_rep, self.free_rows()))  # one control message per rank
            if self.rank == 0:
                all_dec = [b[0] for b in both]
                free = [b[1] for b in both]
                coord.absorb(rnd, all_pre, all_dec)
        return coord.records if self.rank == 0 else None

    # -- control plane (gloo) --------------------------------------------
    def _bcast(self, obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0, group=self.ctrl)
        return box[0]

    def _gather(self, obj):
        out = [None] * self.world if self.rank == 0 else None
        dist.gather_object(obj, out, dst=0, group=self.ctrl)
        return out

    def _allgather(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.ctrl)
        return out


def _slots(chain) -> list[int]:
    """Pool slots of a returned chain: the GPU pool's BlockChain carries them;
    a reference-API pool returns blocks (KVBlock, or plain ids) whose ids the
    backend maps to pages."""
    if hasattr(chain, "slots"):
        return [int(s) for s in chain.slots.tolist()]
    return [int(b) if isinstance(b, (int, np.integer)) else int(b.block_id) for b in chain]


def summarize(records: dict[int, Record], warmup_fraction: float = 0.1) -> dict:
    from .serve import RequestRecord, summarize as _summ
    recs = []
    for r in records.values():
        rr = RequestRecord(r.rid, r.sid, r.model_id, r.issue_us, r.first_token_us, r.done_us, r.out_tokens,
                           r.matched, r.prefilled, r.failed)
        recs.append(rr)
    return _summ(recs, warmup_fraction)


# ------------------------------------------------------------ GPU backends ----

class GpuPrefillBackend(PrefillBackend):
    """A logical prefill worker on this GPU: GPU BlockPool (K7, slot == page),
    its KV pages, PrefillRunner (K1-K3, batched partial prefill)."""

    def __init__(self, cfg, weights, pool_pages: int, max_context: int, max_jobs: int, device: int = 0):
        from .kvstore import BlockPool
        from .model import KVCache, PrefillRunner
        self.cfg = cfg
        self.kv = KVCache(cfg, pool_pages + max_jobs, device)
        self.kv_pages = self.kv.data.view(self.kv.n_pages, -1)
        self.pool = BlockPool(pool_pages, PAGE_TOKENS, device=device, kv_pages=pool_pages,
                              max_query_tokens=max(1 << 16, max_context))
        self.pool_pages, self.max_jobs = pool_pages, max_jobs
        self.runner = PrefillRunner(cfg, weights, self.kv, max_tokens=max_context, device=device)
        self.dev = torch.device("cuda", device)

    def slot_page(self, slot: int) -> int:
        return slot

    def tail_page(self, k: int) -> int:
        if k >= self.max_jobs:
            raise ValueError("more prefill jobs in a round than tail pages")
        return self.pool_pages + k

    def pack(self, pages):
        from .transfer import copy_pages
        buf = torch.empty((len(pages),) + tuple(self.kv_pages.shape[1:]), dtype=self.kv_pages.dtype,
                          device=self.kv_pages.device)
        copy_pages(self.kv_pages, buf, pages, list(range(len(pages))))
        return buf

    def forward(self, seqs) -> None:
        V = self.cfg.vocab
        self.runner.run_batch([(torch.from_numpy((t % V).astype(np.int64)).to(self.dev), p0, pt)
                               for t, p0, pt in seqs], kv_only=True)


class GpuDecodeBackend(DecodeBackend):
    """The decode worker(s) of this GPU: every hosted model's rows in one
    DecodeBatch / CUDA graph (K5/K5-TC GEMV, K6 attention); received context
    pages from a free list, private pages per row."""

    def __init__(self, cfg, modules: dict, rows_per_model: int, ctx_pages: int, max_context: int,
                 max_output: int, device: int = 0):
        from .model import DecodeBatch, DecodeRow, DecodeRunner, KVCache, SessionSpec
        from .transfer import PageAllocator
        self.cfg = cfg
        self.models = sorted(modules)                  # global model indices hosted here
        priv = (max_output + PAGE_TOKENS - 1) // PAGE_TOKENS
        R = len(self.models) * rows_per_model
        self.kv = KVCache(cfg, ctx_pages + R * (1 + priv), device)
        self.kv_pages = self.kv.data.view(self.kv.n_pages, -1)
        self.alloc_ = PageAllocator(0, ctx_pages)
        self.idle_page = ctx_pages                     # valid page for idle rows
        rows, sess = [], []
        nxt = ctx_pages + R
        max_sp = (max_context + PAGE_TOKENS - 1) // PAGE_TOKENS + 1
        for li, m in enumerate(self.models):
            for k in range(rows_per_model):
                rows.append(DecodeRow(module=li, session=len(sess), first_token=0,
                                      pages=list(range(nxt, nxt + priv))))
                nxt += priv
                sess.append(SessionSpec(shared_len=0, pages=[self.idle_page] * max_sp))
        self.batch = DecodeBatch(sess, rows, len(self.models), device)
        self.runner = DecodeRunner(cfg, [modules[m] for m in self.models], self.kv, self.batch, max_output,
                                   device=device)
        self.rows_per_model = rows_per_model
        self.busy = [False] * R
        self.runner.capture()

    def alloc(self, n):
        return self.alloc_.alloc(n)

    def free(self, pages):
        self.alloc_.release(pages)

    def free_row(self, model):
        li = self.models.index(model)
        for k in range(self.rows_per_model):
            r = li * self.rows_per_model + k
            if not self.busy[r]:
                return r
        return None

    def admit(self, row, job, pages):
        # the decode module attends to positions [0, n-1) and processes the
        # last context token itself (model.ts:372-374)
        n = len(job.ctx)
        self.busy[row] = True
        self.batch.update_row(row, n - 1, pages, int(job.ctx[-1] % self.cfg.vocab))

    def retire(self, row):
        self.busy[row] = False
        self.batch.update_row(row, 0, [self.idle_page], 0)

    def step(self):
        self.runner.graph.replay()

    def mark(self):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def resolve(self, marks):
        marks[-1].synchronize()
        t_end = time.perf_counter()
        return [t_end - m.elapsed_time(marks[-1]) / 1e3 for m in marks]

    def copy_pages(self, src, src_pages, dst_pages):
        from .transfer import copy_pages
        copy_pages(src, self.kv_pages, src_pages, dst_pages)

    def unpack(self, buf, pages):
        from .transfer import copy_pages
        copy_pages(buf, self.kv_pages, list(range(len(pages))), pages)
