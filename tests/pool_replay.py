"""Replay the reference-generated pool op streams (tests/golden) through any
pool implementation and compare every observable with the reference's."""

from __future__ import annotations

import gzip
import hashlib
import json
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def load_streams() -> list[dict]:
    return json.loads(gzip.decompress((GOLDEN / "pool_streams.json.gz").read_bytes()))["streams"]


@lru_cache(maxsize=1)
def load_des_logs() -> list[dict]:
    """Pool call logs recorded at the reference's own seam: prefillsim.cluster
    Simulation runs of configs/fast_react.toml (tests/golden/make_golden.py,
    des_call_logs)."""
    return json.loads(gzip.decompress((GOLDEN / "des_pool_log.json.gz").read_bytes()))["streams"]


def expand_tokens(op) -> tuple:
    if "segs" not in op:
        return tuple(op["tokens"])
    out = []
    for sid, purpose, n in op["segs"]:
        base = ((sid + 1) << 32) | (purpose << 16)
        out.extend(base | i for i in range(n))
    return tuple(out)


def digest(rows) -> str:
    rows = sorted([list(r[:2]) + [list(r[2])] + list(r[3:]) for r in rows])
    return hashlib.sha1(json.dumps(rows, separators=(",", ":")).encode()).hexdigest()


class OracleAdapter:
    def __init__(self, capacity, block_size):
        from oracle.pool import OraclePool, OracleCapacityExhausted
        self.p = OraclePool(capacity, block_size)
        self.cap_exc = OracleCapacityExhausted

    def lookup(self, ns, q, now):
        ids = self.p.lookup(ns, q, now)
        return len(ids) * self.p.block_size, ids, ids

    def insert(self, ns, q, now):
        ids = self.p.insert(ns, q, now)
        return ids, ids

    def pin(self, h, now):
        self.p.pin(h, now)

    def release(self, h):
        self.p.release(h)

    def evict(self, need):
        return self.p.evict_until(need)

    def concat(self, handles):
        return [b for h in handles for b in h]

    def counters(self):
        p = self.p
        return p.used_blocks, p.eviction_count, p.matched_tokens, p.lookup_tokens

    def rows(self):
        return self.p.state()

    def footprints(self):
        return dict(self.p.footprint), dict(self.p.peak)


class GpuAdapter:
    def __init__(self, capacity, block_size):
        from paper_2602_12029_b200.kvstore import BlockPool, CapacityExhausted
        self.p = BlockPool(capacity, block_size)
        self.cap_exc = CapacityExhausted

    def lookup(self, ns, q, now):
        m, chain = self.p.longest_prefix_match(ns, q, now)
        return m, chain.ids.tolist(), chain

    def insert(self, ns, q, now):
        chain = self.p.insert(ns, q, now)
        return chain.ids.tolist(), chain

    def pin(self, h, now):
        self.p.pin(h, now)

    def release(self, h):
        self.p.release(h)

    def evict(self, need):
        return self.p.evict_until(need)

    def concat(self, handles):
        # the matched chain extended in place by the allocation (cluster.py:347)
        from paper_2602_12029_b200.kvstore import BlockChain
        out = BlockChain(self.p, handles[0].slots, handles[0].ids)
        for h in handles[1:]:
            out.extend(h)
        return out

    def counters(self):
        p = self.p
        return p.used_blocks, p.eviction_count, p.matched_tokens, p.lookup_tokens

    def rows(self):
        return sorted((b.block_id, b.namespace, b.token_span, b.parent_id, b.ref_count,
                       b.last_access, b.child_count) for b in self.p._blocks.values())

    def footprints(self):
        return self.p.footprint_tokens(), self.p.peak_footprint_tokens()


def _arg(a, handles, op):
    """pin / release argument: one earlier result (ref) or the concatenation
    of several (refs: the DES's matched chain + its allocation)."""
    if "ref" in op:
        return handles[op["ref"]]
    hs = [handles[r] for r in op["refs"]]
    return hs[0] if len(hs) == 1 else a.concat(hs)


def replay(stream: dict, adapter_cls, check_digest_every: int = 1) -> None:
    a = adapter_cls(stream["capacity"], stream["block_size"])
    handles: dict[int, object] = {}
    for i, (op, want) in enumerate(zip(stream["ops"], stream["expect"])):
        kind = op["op"]
        handles[i] = []
        err = None
        got: dict = {}
        try:
            if kind == "lookup":
                m, ids, h = a.lookup(op["ns"], expand_tokens(op), op["now"])
                handles[i] = h
                got = {"matched": m, "ids": ids}
            elif kind == "insert":
                ids, h = a.insert(op["ns"], expand_tokens(op), op["now"])
                handles[i] = h
                got = {"ids": ids}
            elif kind == "pin":
                a.pin(_arg(a, handles, op), op["now"])
            elif kind == "release":
                a.release(_arg(a, handles, op))
            elif kind == "evict":
                got = {"evicted": a.evict(op["need"])}
        except a.cap_exc:
            err = "capacity"
        except RuntimeError:
            err = "underflow"
        ctx = f"{stream['name']} op#{i} {kind}"
        assert err == want["error"], f"{ctx}: error {err} != {want['error']}"
        for k, v in got.items():
            if err is None:
                assert v == want[k], f"{ctx}: {k} {v} != {want[k]}"
        used, ev, mt, lt = a.counters()
        assert (used, ev, mt, lt) == (want["used"], want["evictions"], want["matched_tokens"],
                                      want["lookup_tokens"]), f"{ctx}: counters"
        if check_digest_every and (i % check_digest_every == 0 or i == len(stream["ops"]) - 1) \
                and "digest" in want:
            assert digest(a.rows()) == want["digest"], f"{ctx}: block state differs"
    if "final" in stream:
        rows = [list(r[:2]) + [list(r[2])] + list(r[3:]) for r in a.rows()]
        assert rows == stream["final"], f"{stream['name']}: final state"
    fp, pk = a.footprints()
    assert fp == stream["footprint"] and pk == stream["peak"], f"{stream['name']}: footprints"
    return a
