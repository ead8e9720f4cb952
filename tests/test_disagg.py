"""Prefill/decode disaggregation (disagg.py) on CPU: world_size 3 over gloo,
the reference request life cycle with synthetic backends that write each
position's token id into its KV slot, so every decode admission checks that
the handoff delivered exactly the full context (cached prefix + new tokens +
tail page) to the model's decode rank. Covers cross-rank P2P handoffs, a
same-rank handoff (copy), both serving modes, and the pool oracle as the
prefill workers' block pool."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_12029_b200.disagg import DecodeBackend, PrefillBackend

PT = 16


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _OraclePoolAPI:
    """Reference BlockPool API (kvstore.py:123-250) over the CPU oracle."""

    def __init__(self, cap):
        from oracle.pool import OracleCapacityExhausted, OraclePool
        self.p = OraclePool(cap, PT)
        self.CapacityError = OracleCapacityExhausted

    def longest_prefix_match(self, ns, q, now):
        ids = self.p.lookup(ns, q, now)
        return len(ids) * PT, ids

    def insert(self, ns, q, now):
        return self.p.insert(ns, q, now)

    def pin(self, ids, now):
        self.p.pin(ids, now)

    def release(self, ids):
        self.p.release(ids)


class _FakePrefill(PrefillBackend):
    def __init__(self, max_jobs=64, pages=4096):
        from paper_2602_12029_b200.disagg import PrefillBackend  # noqa: F401
        self.pool = _OraclePoolAPI(pages)
        self.kv_pages = torch.full((pages + max_jobs, PT), -1, dtype=torch.int64)
        self.page_of = {}
        self.pages, self.max_jobs = pages, max_jobs

    def slot_page(self, bid):
        if bid not in self.page_of:
            self.page_of[bid] = len(self.page_of)
        return self.page_of[bid]

    def tail_page(self, k):
        return self.pages + k

    def forward(self, seqs):
        for toks, pos0, pt in seqs:
            for i, t in enumerate(toks):
                p = pos0 + i
                self.kv_pages[pt[p // PT], p % PT] = int(t)


class _FakeDecode(DecodeBackend):
    def __init__(self, models, rows, ctx_pages=4096):
        from paper_2602_12029_b200.transfer import PageAllocator
        self.kv_pages = torch.full((ctx_pages, PT), -2, dtype=torch.int64)
        self.alloc_ = PageAllocator(0, ctx_pages)
        self.models, self.rows = sorted(models), rows
        self.busy = [False] * (len(self.models) * rows)
        self.checked = 0
        self.bad = 0
        self.per_model = {}

    def alloc(self, n):
        return self.alloc_.alloc(n)

    def free(self, pages):
        self.alloc_.release(pages)

    def free_row(self, model):
        li = self.models.index(model)
        for k in range(self.rows):
            r = li * self.rows + k
            if not self.busy[r]:
                return r
        return None

    def admit(self, row, job, pages):
        self.busy[row] = True
        got = self.kv_pages[pages].reshape(-1)[:len(job.ctx)].numpy()
        self.checked += 1
        self.per_model[job.model] = self.per_model.get(job.model, 0) + 1
        if not np.array_equal(got, job.ctx):
            self.bad += 1

    def retire(self, row):
        self.busy[row] = False

    def step(self):
        pass

    def copy_pages(self, src, src_pages, dst_pages):
        for s, d in zip(src_pages, dst_pages):
            self.kv_pages[d].copy_(src[s])


def _placement(mode, world):
    from paper_2602_12029_b200.router import Placement, ServingMode
    if world == 3:
        if mode is ServingMode.PREFILLSHARE:
            return Placement((0, 1), (2, 2, 1, 1))      # 2 shared prefill workers
        return Placement((0, 0, 1, 1), (2, 2, 1, 1))    # one prefill worker per model
    # world 4: rank 0 prefills only; decode replicas 1:many (models 0 and 3
    # on two ranks each), rank 3 also hosts a prefill worker
    reps = ((1, 2), (3,), (1,), (2, 3))
    if mode is ServingMode.PREFILLSHARE:
        return Placement((0, 3), (1, 3, 1, 2), reps)
    return Placement((0, 0, 3, 3), (1, 3, 1, 2), reps)


def _worker(rank, port, mode_name, q, world=3):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_12029_b200 import workload as wl
        from paper_2602_12029_b200.disagg import Coordinator, DisaggServer, summarize
        from paper_2602_12029_b200.router import Router, ServingMode
        mode = ServingMode(mode_name)
        models = list(wl.DEFAULT_MODELS)
        place = _placement(mode, world)
        mine = [w for w, r in enumerate(place.prefill_gpus) if r == rank]
        prefill = {w: _FakePrefill() for w in mine}
        hosted = place.decode_models_on(rank)
        decode = _FakeDecode(hosted, rows=3) if hosted else None
        srv = DisaggServer(place, models, mode, prefill, decode, rows_per_model=3)
        coord = None
        if rank == 0:
            sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=6.0, duration_s=1.0,
                                                     seed=2, turns=2))
            coord = Coordinator(sessions, models, Router(mode, models), place, time_scale=0.02,
                                steps_per_round=48)
        recs = srv.run(coord, max_rounds=5000)
        out = {"rank": rank, "checked": decode.checked if decode else 0, "bad": decode.bad if decode else 0,
               "per_model": decode.per_model if decode else {}, "handoff": srv.handoff_stats()}
        if rank == 0:
            out["n_req"] = sum(s.total_requests for s in sessions)
            out["summary"] = summarize(recs)
            out["done"] = sum(1 for r in recs.values() if r.done_us is not None)
            out["failed"] = sum(1 for r in recs.values() if r.failed)
            out["matched"] = sum(r.matched for r in recs.values())
        q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["prefillshare", "baseline"])
def test_disaggregated_serving_gloo_three_ranks(mode):
    by = _spawn(mode, 3)
    assert by[1]["checked"] > 0 and by[2]["checked"] > 0   # same-rank and cross-rank handoffs


@pytest.mark.parametrize("mode", ["prefillshare", "baseline"])
def test_decode_replicas_gloo_four_ranks(mode):
    """1:many placement: models 0 and 3 have decode replicas on two ranks;
    the coordinator spreads their requests over both replicas (most free
    rows), every context arrives intact, rank 0 (prefill only) decodes
    nothing."""
    by = _spawn(mode, 4)
    assert by[0]["checked"] == 0
    assert by[1]["per_model"].get(0, 0) > 0 and by[2]["per_model"].get(0, 0) > 0
    assert by[2]["per_model"].get(3, 0) > 0 and by[3]["per_model"].get(3, 0) > 0


def _spawn(mode, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, mode, q, world)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(60)
    assert all(p.exitcode == 0 for p in ps)
    by = {r["rank"]: r for r in res}
    r0 = by[0]
    assert r0["done"] == r0["n_req"] and r0["failed"] == 0
    checked = sum(r["checked"] for r in res)
    # every admitted context's pages hold exactly its token ids
    assert checked == r0["n_req"] and sum(r["bad"] for r in res) == 0
    if mode == "prefillshare":
        assert r0["matched"] > 0                             # later agents hit the shared prefix
    assert sum(r["handoff"]["bytes"] for r in res) > 0      # packed cross-rank messages moved
    return by
