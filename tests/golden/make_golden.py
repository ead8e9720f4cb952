"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src); the fixtures it writes are committed and are all
the GPU box ever sees.

    python tests/golden/make_golden.py

pool_streams.json.gz — seeded op streams (lookup / insert / pin / release /
  evict_until, incl. capacity failures and release underflow) replayed
  through prefillsim.kvstore.BlockPool, with the observable outcome of every
  op and a digest of the full block state after every op.
router_traces.json — prefillsim.router.Router decisions over seeded request
  streams in both serving modes.
workload.json — splitmix64 vectors, mix_seed, synth_tokens and a generated
  session list (prefillsim.workload).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def state_digest(blocks) -> str:
    """Canonical digest of a pool's block records (shared with the tests)."""
    rows = sorted(
        (b.block_id, b.namespace, list(b.token_span), b.parent_id, b.ref_count,
         b.last_access, b.child_count)
        for b in blocks
    )
    return hashlib.sha1(json.dumps(rows, separators=(",", ":")).encode()).hexdigest()


def run_stream(BlockPool, CapacityExhausted, capacity, block_size, ops):
    pool = BlockPool(capacity_blocks=capacity, block_size=block_size)
    results = {}  # op index -> blocks returned (reference objects)
    expect = []
    for i, op in enumerate(ops):
        kind = op["op"]
        rec: dict = {}
        results[i] = []  # a failed insert returns nothing to pin/release
        try:
            if kind == "lookup":
                matched, blocks = pool.longest_prefix_match(op["ns"], tuple(expand_tokens(op)), op["now"])
                results[i] = blocks
                rec["matched"] = matched
                rec["ids"] = [b.block_id for b in blocks]
            elif kind == "insert":
                new = pool.insert(op["ns"], tuple(expand_tokens(op)), op["now"])
                results[i] = new
                rec["ids"] = [b.block_id for b in new]
            elif kind == "pin":
                pool.pin(results[op["ref"]], op["now"])
            elif kind == "release":
                pool.release(results[op["ref"]])
            elif kind == "evict":
                rec["evicted"] = pool.evict_until(op["need"])
            rec["error"] = None
        except CapacityExhausted:
            rec["error"] = "capacity"
        except RuntimeError:
            rec["error"] = "underflow"
        rec["used"] = pool.used_blocks
        rec["evictions"] = pool.eviction_count
        rec["matched_tokens"] = pool.matched_tokens
        rec["lookup_tokens"] = pool.lookup_tokens
        rec["digest"] = state_digest(pool._blocks.values())
        expect.append(rec)
    final = sorted(
        (b.block_id, b.namespace, list(b.token_span), b.parent_id, b.ref_count,
         b.last_access, b.child_count)
        for b in pool._blocks.values()
    )
    return expect, final, pool.footprint_tokens(), pool.peak_footprint_tokens(), pool.dump_tree()


def small_random_stream(rng: random.Random):
    """Shape of test_kvstore.py:160-217 (hypothesis op streams)."""
    ops = []
    held = []
    now = 0
    for _ in range(rng.randint(1, 60)):
        now += 1
        ns = rng.choice(["shared", "model:m0", "model:m1"])
        toks = [rng.randint(0, 7) for _ in range(rng.randint(0, 24))]
        if rng.random() < 0.5:
            ops.append({"op": "lookup", "ns": ns, "tokens": toks, "now": now})
            held.append(len(ops) - 1)
            if len(held) > 3:
                ops.append({"op": "release", "ref": held.pop(0)})
        else:
            ops.append({"op": "insert", "ns": ns, "tokens": toks, "now": now})
            if rng.random() < 0.3:
                ops.append({"op": "pin", "ref": len(ops) - 1, "now": now})
                held.append(len(ops) - 2)
    return ops


def a2_stream(rng: random.Random, block_size: int, n_ops: int):
    """Shape of test_acceptance.py:283-324 (A2 randomized equivalence)."""
    ops = []
    held = []
    for now in range(n_ops):
        ns = rng.choice(["shared", "model:a", "model:b"])
        base = rng.randrange(6)
        length = rng.randrange(0, 4 * block_size + 3)
        toks = [base * 1000 + t for t in range(length)]
        if rng.random() < 0.5:
            ops.append({"op": "lookup", "ns": ns, "tokens": toks, "now": now})
            held.append(len(ops) - 1)
        else:
            ops.append({"op": "insert", "ns": ns, "tokens": toks, "now": now})
        while len(held) > rng.randrange(1, 5):
            ops.append({"op": "release", "ref": held.pop(0)})
    return ops


def expand_tokens(op) -> list:
    """Token list of an op; DES ops store synth_tokens segments
    (workload.py:375-387 packing) instead of the expanded ids."""
    if "segs" not in op:
        return op["tokens"]
    out = []
    for sid, purpose, n in op["segs"]:
        base = ((sid + 1) << 32) | (purpose << 16)
        out.extend(base | i for i in range(n))
    return out


def des_like_stream(rng: random.Random, wl, n_sessions: int, turns: int):
    """Multi-turn agent contexts of synth_tokens ids (cluster.py:271-366
    order: lookup at prefill start, insert + pin at prefill complete, release
    at handoff) with interleaved sessions and eviction pressure."""
    ops = []
    segs = {s: [[s, 0, 512]] for s in range(n_sessions)}
    step = {s: 0 for s in range(n_sessions)}
    now = 0
    pending = []
    for _ in range(n_sessions * turns):
        s = rng.randrange(n_sessions)
        segs[s].append([s, 2 * step[s] + 1, 64])
        now += rng.randint(1, 1000)
        ops.append({"op": "lookup", "ns": "shared", "segs": [list(x) for x in segs[s]], "now": now})
        lk = len(ops) - 1
        now += rng.randint(1, 1000)
        ops.append({"op": "insert", "ns": "shared", "segs": [list(x) for x in segs[s]], "now": now})
        ins = len(ops) - 1
        ops.append({"op": "pin", "ref": ins, "now": now})
        pending.append((lk, ins))
        segs[s].append([s, 2 * step[s] + 2, 128])
        step[s] += 1
        while len(pending) > rng.randint(0, 3):
            a, b = pending.pop(0)
            ops.append({"op": "release", "ref": a})
            ops.append({"op": "release", "ref": b})
    for a, b in pending:
        ops.append({"op": "release", "ref": a})
        ops.append({"op": "release", "ref": b})
    ops.append({"op": "evict", "need": 10})
    return ops


def underflow_stream():
    return [
        {"op": "insert", "ns": "ns", "tokens": [1, 2, 3, 4, 5, 6, 7, 8], "now": 1},
        {"op": "pin", "ref": 0, "now": 2},
        {"op": "lookup", "ns": "ns", "tokens": [1, 2, 3, 4], "now": 3},
        {"op": "release", "ref": 0},
        {"op": "release", "ref": 0},          # underflow at the first block
        {"op": "release", "ref": 2},
        {"op": "release", "ref": 2},          # underflow
        {"op": "evict", "need": 3},           # need > capacity
        {"op": "evict", "need": 2},
    ]


def pool_fixtures(wl, BlockPool, CapacityExhausted):
    rng = random.Random(20260212)
    streams = []
    for i in range(60):
        bs = rng.choice([1, 2, 4])
        cap = rng.randint(1, 12)
        ops = small_random_stream(rng)
        streams.append({"name": f"small_{i}", "capacity": cap, "block_size": bs, "ops": ops})
    for bs in (1, 4, 16):
        ops = a2_stream(random.Random(1000 + bs), bs, 1200)
        streams.append({"name": f"a2_bs{bs}", "capacity": 48, "block_size": bs, "ops": ops})
    streams.append({"name": "des_pressure", "capacity": 300, "block_size": 16,
                    "ops": des_like_stream(random.Random(7), wl, 12, 30)})
    streams.append({"name": "des_unbounded", "capacity": 1 << 62, "block_size": 16,
                    "ops": des_like_stream(random.Random(8), wl, 8, 12)})
    streams.append({"name": "underflow", "capacity": 2, "block_size": 4, "ops": underflow_stream()})
    for st in streams:
        expect, final, fp, peak, dump = run_stream(BlockPool, CapacityExhausted, st["capacity"],
                                                   st["block_size"], st["ops"])
        st["expect"] = expect
        st["final"] = final
        st["footprint"] = fp
        st["peak"] = peak
        st["dump_tree"] = dump
    return streams


def _compress_tokens(toks) -> dict:
    """Packed synthetic ids (workload.py:142-154) as [sid, purpose, n] runs
    when the context is made of whole segments from index 0, else raw."""
    segs, i, n = [], 0, len(toks)
    while i < n:
        t = toks[i]
        sid, purpose, idx = (t >> 32) - 1, (t >> 16) & 0xFFFF, t & 0xFFFF
        if idx != 0 or sid < 0:
            return {"tokens": list(toks)}
        j = i
        while j < n and toks[j] == (((sid + 1) << 32) | (purpose << 16) | (j - i)):
            j += 1
        segs.append([sid, purpose, j - i])
        i = j
    return {"segs": segs}


def des_call_logs(runs=((7500, "baseline"), (7500, "prefillshare"), (1500, "baseline"),
                        (1500, "prefillshare"), (100, "prefillshare"))):
    """The REAL call pattern at the drop-in seam (cluster.py:30):
    run prefillsim.cluster.Simulation on configs/fast_react.toml (60 s ReAct
    workload, the reference fleet) in both modes, with prefillsim.cluster's
    BlockPool replaced by a recording subclass. Every pool op of every
    prefill worker is logged in the pool-stream format (pin / release
    reference the lookup / insert results they were given: release gets the
    matched chain extended in place by the allocation, cluster.py:330, 347,
    409), with the reference's outcome, counters and a state digest every
    25 ops. Runs with 1500- and 100-block pools add eviction pressure and
    capacity failures (contexts longer than the pool: CapacityExhausted,
    caught by class, cluster.py:348). The recorded run's report is checked to be identical to an
    unrecorded run's (the subclass does not perturb the simulation)."""
    import dataclasses

    from prefillsim import cluster, config as pconfig, experiment, kvstore
    base_cfg = pconfig.load_config("/root/reference/pkg/configs/fast_react.toml")
    logs = []
    for cap, mode in runs:
        if True:
            cfg = dataclasses.replace(base_cfg, run=dataclasses.replace(base_cfg.run, mode=mode),
                                      cache=dataclasses.replace(base_cfg.cache, prefill_capacity_blocks=cap))
            _, plain = experiment.run_once(cfg)
            pools = []

            class RecordingPool(kvstore.BlockPool):
                def __init__(self, capacity_blocks, block_size):
                    super().__init__(capacity_blocks, block_size)
                    self.log, self.expect = [], []
                    # id(list returned by lookup / insert) -> (op index, the list): the
                    # list is kept alive so its id is never reused by a later list
                    self.obj_op = {}
                    self.ins_op = {}
                    pools.append(self)

                def _record(self, op, res, err):
                    rec = {"error": err, "used": self.used_blocks, "evictions": self.eviction_count,
                           "matched_tokens": self.matched_tokens, "lookup_tokens": self.lookup_tokens}
                    rec.update(res)
                    if len(self.log) % 25 == 0:
                        rec["digest"] = state_digest(self._blocks.values())
                    self.log.append(op)
                    self.expect.append(rec)

                def _refs(self, blocks):
                    if id(blocks) in self.ins_op:  # pin(allocated), cluster.py:346
                        return [self.ins_op[id(blocks)][0]]
                    # release(matched chain extended in place by the allocation), cluster.py:347, 349, 409
                    i = self.obj_op[id(blocks)][0]
                    n0 = len(self.expect[i]["ids"])
                    refs = [i]
                    if len(blocks) > n0:
                        tail = [b.block_id for b in blocks[n0:]]
                        refs.append(next(k for k in range(len(self.log) - 1, i, -1)
                                         if self.log[k]["op"] == "insert" and self.expect[k].get("ids") == tail))
                    return refs

                def longest_prefix_match(self, ns, query, now):
                    m, blocks = super().longest_prefix_match(ns, query, now)
                    i = len(self.log)
                    self.obj_op[id(blocks)] = (i, blocks)
                    self._record(dict({"op": "lookup", "ns": ns, "now": now}, **_compress_tokens(query)),
                                 {"matched": m, "ids": [b.block_id for b in blocks]}, None)
                    return m, blocks

                def insert(self, ns, seq, now):
                    op = dict({"op": "insert", "ns": ns, "now": now}, **_compress_tokens(seq))
                    try:
                        new = super().insert(ns, seq, now)
                    except kvstore.CapacityExhausted:
                        self._record(op, {}, "capacity")
                        raise
                    self.ins_op[id(new)] = (len(self.log), new)
                    self._record(op, {"ids": [b.block_id for b in new]}, None)
                    return new

                def pin(self, blocks, now):
                    refs = self._refs(blocks)
                    super().pin(blocks, now)
                    self._record({"op": "pin", "refs": refs, "now": now}, {}, None)

                def release(self, blocks):
                    refs = self._refs(blocks)
                    super().release(blocks)
                    self._record({"op": "release", "refs": refs}, {}, None)

            saved = cluster.BlockPool
            cluster.BlockPool = RecordingPool
            try:
                _, rec_report = experiment.run_once(cfg)
            finally:
                cluster.BlockPool = saved
            assert json.dumps(rec_report, sort_keys=True) == json.dumps(plain, sort_keys=True)
            for w, pool in enumerate(pools):
                final = sorted(
                    (b.block_id, b.namespace, list(b.token_span), b.parent_id, b.ref_count,
                     b.last_access, b.child_count)
                    for b in pool._blocks.values())
                pool.expect[-1]["digest"] = state_digest(pool._blocks.values())
                # (the full final state is covered by the last op's digest;
                # dump_tree kept for worker 0)
                del final
                logs.append({"name": f"des_fast_react_{mode}_cap{cap}_w{w}", "capacity": cap,
                             "block_size": pool.block_size, "ops": pool.log, "expect": pool.expect,
                             "footprint": dict(pool.footprint_tokens()),
                             "peak": dict(pool.peak_footprint_tokens()),
                             **({"dump_tree": pool.dump_tree()} if w == 0 else {}),
                             "report": {k: plain[k] for k in ("prefix_hit_ratio", "eviction_count",
                                                              "failure_count", "request_count")}})
    return logs


def check_logs_replay(logs, kvstore):
    """Self-check of the recorded logs: replayed through a fresh reference
    BlockPool with the tests' replay harness, every outcome and digest must
    reproduce (catches a wrongly resolved pin / release argument)."""
    sys.path.insert(0, str(OUT.parent))
    import pool_replay as pr

    class RefAdapter:
        def __init__(self, cap, bs):
            self.p = kvstore.BlockPool(cap, bs)
            self.cap_exc = kvstore.CapacityExhausted

        def lookup(self, ns, q, now):
            m, b = self.p.longest_prefix_match(ns, q, now)
            return m, [x.block_id for x in b], b

        def insert(self, ns, q, now):
            b = self.p.insert(ns, q, now)
            return [x.block_id for x in b], b

        def pin(self, h, now):
            self.p.pin(h, now)

        def release(self, h):
            self.p.release(h)

        def concat(self, hs):
            return [b for h in hs for b in h]

        def counters(self):
            p = self.p
            return p.used_blocks, p.eviction_count, p.matched_tokens, p.lookup_tokens

        def rows(self):
            return sorted((b.block_id, b.namespace, b.token_span, b.parent_id, b.ref_count, b.last_access,
                           b.child_count) for b in self.p._blocks.values())

        def footprints(self):
            return self.p.footprint_tokens(), self.p.peak_footprint_tokens()
    for st in logs:
        pr.replay(st, RefAdapter, check_digest_every=25)


def router_fixtures(core, router):
    rng = random.Random(99)
    models = ["model_a", "model_b", "model_c", "model_d"]
    traces = []
    for mode in (router.ServingMode.BASELINE, router.ServingMode.PREFILLSHARE):
        r = router.Router(mode, models)
        steps = []
        for i in range(400):
            sid = rng.randrange(60)
            m = rng.choice(models + (["model_x"] if rng.random() < 0.02 else []))
            depths = [rng.randrange(6) for _ in range(4)]
            req = core.Request(request_id=i, session_id=sid, model_id=m, context_snapshot=(),
                               output_len=1, issue_time=0)
            try:
                w = r.route_prefill(req, depths)
                d = r.decode_worker(req)
                steps.append({"session": sid, "model": m, "depths": depths, "prefill": w,
                              "decode": d, "ns": r.prefill_namespace(m)})
            except router.ConfigurationError:
                steps.append({"session": sid, "model": m, "depths": depths, "error": "config"})
        traces.append({"mode": mode.value, "models": models, "steps": steps})
    return traces


def sweep_fixtures():
    """experiment.py's sweep protocol: per-cell workload seeds of both axes
    and the sweep table of synthetic cells (incl. auto-concurrency cells)."""
    import dataclasses

    from prefillsim import config as pconfig, experiment
    cfg = pconfig.load_config("/root/reference/pkg/configs/fast_react.toml")
    cfg = dataclasses.replace(cfg, run=dataclasses.replace(cfg.run, seed=7))
    seeds = []
    for axis, values in (("arrival_rate", [0.5, 1, 2, 4, 8, 16.25]), ("max_concurrent_sessions", [10, 20, 160])):
        for v in values:
            c = experiment._cell_config(cfg, axis, v)
            seeds.append({"axis": axis, "value": v, "seed": str(c.run.seed),
                          "rate": c.workload.arrival_rate_per_s, "cap": c.run.max_concurrent_sessions})
    cells, spec = [], []
    for i, (axis, value, mode, cap, chosen) in enumerate([
            ("arrival_rate", 4.0, "baseline", 0, 40), ("arrival_rate", 4.0, "prefillshare", 0, 160),
            ("max_concurrent_sessions", 20, "prefillshare", 20, None),
            ("max_concurrent_sessions", 160, "baseline", 160, None)]):
        rep = {"config": {"run": {"max_concurrent_sessions": cap}}, "throughput_tok_per_s": 1234.5678 * (i + 1),
               "p95_e2e_us": None if i == 3 else 1000 * (i + 7), "mean_ttft_us": None if i == 2 else 12.25 * i,
               "prefix_hit_ratio": 0.8627450980392157 / (i + 1), "failure_count": i}
        cells.append(experiment.SweepCell(axis=axis, value=float(value), mode=mode, report=rep, chosen_cap=chosen))
        spec.append({"axis": axis, "value": value, "mode": mode, "cap": cap, "chosen_cap": chosen, "report": rep})
    return {"cell_seeds": seeds, "table_cells": spec, "table": experiment.sweep_table(cells),
            "cap_grid": list(experiment.DEFAULT_CAP_GRID)}


def workload_fixtures(wl):
    s = wl.splitmix64(0)
    vec = [next(s) for _ in range(8)]
    cfg = wl.WorkloadConfig(pattern="react", arrival_rate_per_s=4.0, duration_s=20.0, seed=3)
    sessions = json.loads(wl.export_sessions(wl.generate(cfg)))
    return {
        "splitmix64_seed0": [str(v) for v in vec],
        "mix_seed": {"1,2": str(wl.mix_seed(1, 2)), "0": str(wl.mix_seed(0)),
                     "0,0": str(wl.mix_seed(0, 0))},
        "synth_tokens_3_5_4": [str(t) for t in wl.synth_tokens(3, 5, 4)],
        "generate_react_seed3_20s": sessions,
    }


def main() -> None:
    sys.path.insert(0, str(REF))
    from prefillsim import core, kvstore, router, workload as wl  # noqa: E402

    pools = pool_fixtures(wl, kvstore.BlockPool, kvstore.CapacityExhausted)
    blob = json.dumps({"generator": "prefillsim.kvstore.BlockPool", "streams": pools},
                      separators=(",", ":")).encode()
    (OUT / "pool_streams.json.gz").write_bytes(gzip.compress(blob, 9, mtime=0))
    (OUT / "router_traces.json").write_text(json.dumps(router_fixtures(core, router)))
    logs = des_call_logs()
    check_logs_replay(logs, kvstore)
    blob = json.dumps({"generator": "prefillsim.cluster.Simulation + recording prefillsim.kvstore.BlockPool "
                                    "(configs/fast_react.toml)", "streams": logs},
                      separators=(",", ":")).encode()
    (OUT / "des_pool_log.json.gz").write_bytes(gzip.compress(blob, 9, mtime=0))
    wf = workload_fixtures(wl)
    wf["sweep"] = sweep_fixtures()
    (OUT / "workload.json").write_text(json.dumps(wf, indent=0))
    n_ops = sum(len(s["ops"]) for s in pools)
    print(f"pool streams: {len(pools)} ({n_ops} ops); router traces; workload vectors")


if __name__ == "__main__":
    main()
