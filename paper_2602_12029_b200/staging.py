"""Host staging tier behind the GPU prefix pool (the
paper's KV staging under memory pressure).

Under load the shared prefix pool fills up and evicts LRU blocks
(kvstore.py:191-235); a later request of the same session then misses and
the base module recomputes those tokens. The tier keeps a write-through copy
of every computed full block in pinned host memory (LRU over its own
capacity), found by a rolling key of namespace + the block's full token path
(a block's KV is a function of exactly that prefix) and verified by the
block's exact edge (namespace, parent key, 16 tokens) before any reload. On a GPU miss, the pool still allocates
the blocks exactly as the reference does (hit / miss / eviction accounting
is unchanged); the consecutive missing blocks found in the tier are copied
back host -> device into their new pages instead of being recomputed, so the
forward starts after them. Costs: one 2 MiB D2H per computed block (side
stream, overlapped) and one H2D per reloaded block (~40 us at PCIe 5 rates)
versus ~16 tokens of 8B prefill (~0.2 ms) per recomputed block.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np
import torch

from .model import PAGE_TOKENS, KVCache


ROOT_KEY = 0  # parent key of a context's first block


def block_keys(ns: str, ctx: np.ndarray, n_blocks: int) -> list[int]:
    """Rolling key of each full block: hash(namespace, tokens[0, 16(k+1))).
    A key only FINDS a candidate; TierIndex.lookup verifies the candidate's
    exact edge before it is reloaded."""
    keys, h = [], hash(("psk-tier", ns))
    for k in range(n_blocks):
        h = hash((h, ctx[k * PAGE_TOKENS:(k + 1) * PAGE_TOKENS].tobytes()))
        keys.append(h)
    return keys


def block_edges(ns: str, ctx: np.ndarray, keys: list[int], first: int, last: int) -> list[tuple]:
    """Exact identity of blocks [first, last): (namespace, parent block's
    key, the block's 16 tokens) -- the reference's edge key
    (ns, parent, token_span), kvstore.py:69-70."""
    return [(ns, keys[k - 1] if k > 0 else ROOT_KEY, ctx[k * PAGE_TOKENS:(k + 1) * PAGE_TOKENS].tobytes())
            for k in range(first, last)]


class TierIndex:
    """Host-side index of the tier: key -> slot (LRU order) plus each slot's
    exact edge. Lookup walks the context's blocks from the first requested
    one and stops at the first block whose key is absent OR whose stored edge
    (namespace, parent key, 16 tokens) differs from the context's: a 64-bit
    key collision can never reload another path's KV. (By induction from
    the first block: equal tokens at every level and equal parent keys mean
    the stored block's full token path is the context's.)"""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.lru: OrderedDict[int, int] = OrderedDict()  # key -> slot
        self.edge: dict[int, tuple] = {}                 # slot -> (ns, parent key, token bytes)
        self.free = list(range(capacity - 1, -1, -1))
        self.collisions = 0

    def lookup(self, keys: list[int], edges: list[tuple]) -> list[int]:
        out = []
        for k, e in zip(keys, edges):
            s = self.lru.get(k)
            if s is None:
                break
            if self.edge[s] != e:  # same key, different block: a collision
                self.collisions += 1
                break
            self.lru.move_to_end(k)
            out.append(s)
        return out

    def place(self, key: int, edge: tuple) -> int | None:
        """Slot for a new block (None: already present). Evicts the LRU entry
        when full."""
        if key in self.lru:
            self.lru.move_to_end(key)
            return None
        if self.free:
            s = self.free.pop()
        else:
            _, s = self.lru.popitem(last=False)
        self.lru[key] = s
        self.edge[s] = edge
        return s


class HostKVTier:
    def __init__(self, kv: KVCache, capacity_blocks: int):
        self.kv = kv
        self.capacity = capacity_blocks
        self.buf = torch.empty(capacity_blocks, kv.data.shape[1], dtype=kv.data.dtype).pin_memory()
        self.index = TierIndex(capacity_blocks)
        self.d2h = torch.cuda.Stream(device=kv.data.device)
        self.stored = 0
        self.reloaded = 0

    def lookup(self, keys: list[int], edges: list[tuple]) -> list[int]:
        """Host slots of the longest verified run of blocks present
        (LRU-touched); edges from block_edges()."""
        return self.index.lookup(keys, edges)

    def reload(self, slots: list[int], pages: list[int]) -> None:
        """H2D into the pool's new pages, ordered on the current stream (after
        any pending write-through into those host slots)."""
        self.fence()
        for s, p in zip(slots, pages):
            self.kv.data[p].copy_(self.buf[s], non_blocking=True)
        self.reloaded += len(slots)

    def store(self, keys: list[int], edges: list[tuple], pages: list[int]) -> None:
        """Write-through of freshly computed blocks (after the forward that
        wrote them, on a side stream)."""
        cur = torch.cuda.current_stream(self.kv.data.device)
        self.d2h.wait_stream(cur)  # the forward (and any reload reading a slot reused below) is done
        with torch.cuda.stream(self.d2h):
            for k, e, p in zip(keys, edges, pages):
                s = self.index.place(k, e)
                if s is None:
                    continue
                self.buf[s].copy_(self.kv.data[p], non_blocking=True)
                self.stored += 1

    def fence(self) -> None:
        """Order later work on the current stream after the pending D2H copies
        (a page is reused only after its copy landed)."""
        torch.cuda.current_stream(self.kv.data.device).wait_stream(self.d2h)

    def stats(self) -> dict:
        return {"capacity_blocks": self.capacity, "resident_blocks": len(self.index.lru), "stored": self.stored,
                "reloaded": self.reloaded, "key_collisions_rejected": self.index.collisions}


class DecodeResidency:
    """One decode worker's GPU-resident KV budget with staged handoff through
    pinned host memory: the reference's decode-side accounting
    (cluster.py:59-75: capacity_tokens = decode_capacity_blocks x block_size,
    resident fraction) and staging rule (costs.py:66-83, cluster.py:376-394:
    a handoff arriving while the resident fraction exceeds the staging
    threshold is staged), with the data movement vLLM actually does
    (App. B: KV staged in CPU memory, reloaded when the session is
    scheduled).

    Pages [first, first + capacity) of the KV cache belong to this worker.
    take / give account the contexts admitted to the decode batch; stage()
    gathers a context's pages (K8 copy on a side stream, then one D2H into a
    pinned buffer) and reload() brings it back (one H2D, then a K8 scatter
    into freshly taken pages). The bytes are moved, not recomputed: reload
    is bit-exact."""

    def __init__(self, kv: KVCache, first: int, capacity: int, threshold: float = 0.9):
        from .transfer import PageAllocator
        self.kv = kv
        self.pages = kv.data.view(kv.n_pages, -1)
        self.alloc = PageAllocator(first, capacity)
        self.capacity, self.threshold = capacity, threshold
        self.resident = 0
        self.staged_count = 0
        self.staged_bytes = 0
        self.d2h = torch.cuda.Stream(device=kv.data.device)

    def fraction(self) -> float:
        return self.resident / self.capacity if self.capacity > 0 else 0.0

    def must_stage(self, n: int) -> bool:
        """cluster.py:379-381 (fraction > threshold), plus: the context does
        not fit the free budget at all."""
        return self.fraction() > self.threshold or self.resident + n > self.capacity

    def can_take(self, n: int) -> bool:
        return self.resident + n <= self.capacity

    def take(self, n: int) -> list[int]:
        pages = self.alloc.alloc(n)
        self.resident += n
        return pages

    def give(self, pages: list[int]) -> None:
        self.alloc.release(pages)
        self.resident -= len(pages)

    def stage(self, src_pages: list[int]) -> torch.Tensor:
        """Context pages -> pinned host buffer (side stream, after the work
        queued on the current stream that wrote them)."""
        from .transfer import copy_pages
        n = len(src_pages)
        cur = torch.cuda.current_stream(self.kv.data.device)
        host = torch.empty((n, self.pages.shape[1]), dtype=self.pages.dtype).pin_memory()
        self.d2h.wait_stream(cur)
        with torch.cuda.stream(self.d2h):
            tmp = torch.empty((n, self.pages.shape[1]), dtype=self.pages.dtype, device=self.pages.device)
            copy_pages(self.pages, tmp, src_pages, list(range(n)))
            host.copy_(tmp, non_blocking=True)
        self.staged_count += 1
        self.staged_bytes += host.numel() * host.element_size()
        return host

    def reload(self, host: torch.Tensor, pages: list[int]) -> None:
        """Pinned host buffer -> taken pages, ordered on the current stream
        after the staging copy."""
        from .transfer import copy_pages
        self.fence()
        tmp = host.to(self.pages.device, non_blocking=True)
        copy_pages(tmp, self.pages, list(range(len(pages))), pages)

    def fence(self) -> None:
        """Later work on the current stream (which may overwrite the source
        pages of a pending stage) waits for the staging copies."""
        torch.cuda.current_stream(self.kv.data.device).wait_stream(self.d2h)
