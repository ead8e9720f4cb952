"""CPU oracle of the reference KV block pool — TEST INFRASTRUCTURE ONLY.

Restates src/prefillsim/kvstore.py:59-250 without its lazy heap: eviction is
a plain argmin scan over the unpinned leaves keyed (last_access, block_id),
which is what the heap computes (kvstore.py:212-223) and what the reference's
naive tests/reference_pool.py checks. Full record state (ref counts, child
counts, parents) is kept so the GPU pool can be compared field by field.
Pinned against the reference via tests/golden/pool_*.json.
"""

from __future__ import annotations

from dataclasses import dataclass


class OracleCapacityExhausted(Exception):
    pass


@dataclass
class Rec:
    block_id: int
    namespace: str
    token_span: tuple
    parent_id: int
    ref_count: int = 0
    last_access: int = 0
    child_count: int = 0


class OraclePool:
    def __init__(self, capacity_blocks: int, block_size: int) -> None:
        if capacity_blocks < 0 or block_size < 1:
            raise ValueError("capacity_blocks >= 0 and block_size >= 1 required")
        self.capacity_blocks = capacity_blocks
        self.block_size = block_size
        self.recs: dict[int, Rec] = {}
        self.edges: dict[tuple, int] = {}  # (ns, parent_id, span) -> block_id  (kvstore.py:69-70)
        self.next_id = 0
        self.matched_tokens = 0
        self.lookup_tokens = 0
        self.eviction_count = 0
        self.footprint: dict[str, int] = {}
        self.peak: dict[str, int] = {}

    @property
    def used_blocks(self) -> int:
        return len(self.recs)

    def chain(self, ns: str, q: tuple) -> list[int]:
        """kvstore.py:109-121."""
        bs, out, parent = self.block_size, [], -1
        for k in range(len(q) // bs):
            bid = self.edges.get((ns, parent, tuple(q[k * bs:(k + 1) * bs])))
            if bid is None:
                break
            out.append(bid)
            parent = bid
        return out

    def lookup(self, ns: str, q: tuple, now: int) -> list[int]:
        """kvstore.py:123-138."""
        ids = self.chain(ns, q)
        for b in ids:
            self.recs[b].ref_count += 1
            self.recs[b].last_access = now
        self.lookup_tokens += len(q)
        self.matched_tokens += len(ids) * self.block_size
        return ids

    def _victim(self):
        best = None
        for r in self.recs.values():
            if r.ref_count == 0 and r.child_count == 0:
                if best is None or (r.last_access, r.block_id) < (best.last_access, best.block_id):
                    best = r
        return best

    def evict_until(self, need: int) -> int:
        """kvstore.py:191-210 + _evict :225-235."""
        if need > self.capacity_blocks:
            raise OracleCapacityExhausted("need exceeds capacity")
        n = 0
        while self.capacity_blocks - len(self.recs) < need:
            v = self._victim()
            if v is None:
                raise OracleCapacityExhausted("all pinned")
            del self.edges[(v.namespace, v.parent_id, v.token_span)]
            del self.recs[v.block_id]
            self.footprint[v.namespace] -= len(v.token_span)
            self.eviction_count += 1
            n += 1
            if v.parent_id in self.recs:
                self.recs[v.parent_id].child_count -= 1
        return n

    def insert(self, ns: str, q: tuple, now: int) -> list[int]:
        """kvstore.py:140-189."""
        bs = self.block_size
        n_full = len(q) // bs
        ids = self.chain(ns, q)
        need = n_full - len(ids)
        if need == 0:
            return []
        for b in ids:  # protect the matched chain (kvstore.py:153-156)
            self.recs[b].ref_count += 1
        try:
            if self.capacity_blocks - len(self.recs) < need:
                self.evict_until(need)
        finally:
            for b in ids:
                self.recs[b].ref_count -= 1
        parent = ids[-1] if ids else -1
        if ids:
            self.recs[ids[-1]].child_count += 1
        new = []
        for k in range(len(ids), n_full):
            span = tuple(q[k * bs:(k + 1) * bs])
            bid = self.next_id
            self.next_id += 1
            self.recs[bid] = Rec(bid, ns, span, parent, 0, now, 1)
            self.edges[(ns, parent, span)] = bid
            new.append(bid)
            parent = bid
        self.recs[new[-1]].child_count = 0
        self.footprint[ns] = self.footprint.get(ns, 0) + need * bs
        self.peak[ns] = max(self.peak.get(ns, 0), self.footprint[ns])
        return new

    def pin(self, ids: list[int], now: int) -> None:
        for b in ids:
            self.recs[b].ref_count += 1
            self.recs[b].last_access = now

    def release(self, ids: list[int]) -> None:
        for b in ids:
            r = self.recs[b]
            if r.ref_count <= 0:
                raise RuntimeError(f"release underflow on block {b}")
            r.ref_count -= 1

    def state(self) -> list[tuple]:
        """Canonical full state for equality checks."""
        return sorted((r.block_id, r.namespace, r.token_span, r.parent_id, r.ref_count,
                       r.last_access, r.child_count) for r in self.recs.values())
