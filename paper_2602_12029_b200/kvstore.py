"""Drop-in GPU KV block pool behind the reference BlockPool API.

Mirrors src/prefillsim/kvstore.py (BlockPool, KVBlock, PoolStats,
CapacityExhausted, SHARED_NS, model_ns) with the index, refcounts, LRU and
allocator living on the GPU (K7, csrc/pool.cu). Each public op is one kernel
launch plus one stream sync; this module only stages token ids into pinned
memory and wraps results.

Plug-in, as the reference's own seam allows (cluster.py:30, :158):

    import prefillsim.cluster, prefillsim.kvstore
    from paper_2602_12029_b200 import kvstore as gkv
    gkv.BlockPool.CapacityError = prefillsim.kvstore.CapacityExhausted
    prefillsim.cluster.BlockPool = gkv.BlockPool

Differences that are invisible to the reference's callers: blocks are
returned as live handles (BlockRef) inside a BlockChain sequence instead of
Python KVBlock objects; `_blocks` is a snapshot mapping block_id -> KVBlock
read back from the device (tests read it, kvstore.py:211/224 of the
reference tests).
"""

from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass
from typing import Iterable, Iterator, Sequence

import numpy as np

from . import _lib

SHARED_NS = "shared"  # kvstore.py:20


def model_ns(model_id: str) -> str:  # kvstore.py:23-24
    return f"model:{model_id}"


class CapacityExhausted(Exception):
    """Raised when pinned blocks prevent freeing enough space (kvstore.py:27)."""


@dataclass
class KVBlock:
    """Snapshot of one block record (fields of kvstore.py:31-40)."""

    block_id: int
    namespace: str
    token_span: tuple
    ref_count: int = 0
    last_access: int = 0
    parent_id: int = -1
    child_count: int = 0


@dataclass
class PoolStats:  # kvstore.py:43-56
    capacity_blocks: int
    used_blocks: int
    free_blocks: int
    matched_tokens: int
    lookup_tokens: int
    eviction_count: int

    @property
    def hit_ratio(self) -> float:
        if self.lookup_tokens == 0:
            return 0.0
        return self.matched_tokens / self.lookup_tokens


class BlockRef:
    """Live handle to a block on the device (slot + block id). Attribute reads
    fetch the record, so they always reflect the current refcount/access."""

    __slots__ = ("_pool", "slot", "block_id")

    def __init__(self, pool: "BlockPool", slot: int, block_id: int) -> None:
        self._pool = pool
        self.slot = int(slot)
        self.block_id = int(block_id)

    def _rec(self):
        return self._pool._read_record(self.slot, self.block_id)

    @property
    def namespace(self) -> str:
        return self._pool._ns_name(self._rec()[0][2])

    @property
    def token_span(self) -> tuple:
        return self._rec()[1]

    @property
    def ref_count(self) -> int:
        return self._rec()[0][3]

    @property
    def child_count(self) -> int:
        return self._rec()[0][4]

    @property
    def last_access(self) -> int:
        return self._rec()[0][5]

    @property
    def parent_id(self) -> int:
        return self._rec()[0][1]

    def __eq__(self, other) -> bool:
        return isinstance(other, BlockRef) and other.block_id == self.block_id and other._pool is self._pool

    def __hash__(self) -> int:
        return hash((id(self._pool), self.block_id))

    def __repr__(self) -> str:
        return f"BlockRef(block_id={self.block_id}, slot={self.slot})"


class BlockChain(Sequence):
    """Array-backed list of block handles (what lookup/insert return).

    Supports the list operations the reference's callers use on the returned
    lists (iteration, len, indexing, ==, extend — cluster.py:347)."""

    def __init__(self, pool: "BlockPool", slots: np.ndarray, ids: np.ndarray) -> None:
        self._pool = pool
        self.slots = np.ascontiguousarray(slots, dtype=np.int32)
        self.ids = np.ascontiguousarray(ids, dtype=np.int64)

    def __len__(self) -> int:
        return len(self.ids)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return BlockChain(self._pool, self.slots[i], self.ids[i])
        return BlockRef(self._pool, self.slots[i], self.ids[i])

    def __iter__(self) -> Iterator[BlockRef]:
        for s, b in zip(self.slots.tolist(), self.ids.tolist()):
            yield BlockRef(self._pool, s, b)

    def __eq__(self, other) -> bool:
        if isinstance(other, BlockChain):
            return bool(np.array_equal(self.ids, other.ids))
        if isinstance(other, (list, tuple)):
            return len(other) == len(self) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def extend(self, other: Iterable) -> None:
        s, b = _handles_of(other)
        self.slots = np.concatenate([self.slots, s])
        self.ids = np.concatenate([self.ids, b])

    def append(self, ref: BlockRef) -> None:
        self.extend([ref])

    def __iadd__(self, other):
        self.extend(other)
        return self

    def __repr__(self) -> str:
        return f"BlockChain(ids={self.ids.tolist()})"


def _handles_of(blocks) -> tuple[np.ndarray, np.ndarray]:
    if isinstance(blocks, BlockChain):
        return blocks.slots, blocks.ids
    refs = list(blocks)
    for r in refs:
        if not isinstance(r, BlockRef):
            raise TypeError(f"not a GPU block handle: {r!r}")
    return (np.fromiter((r.slot for r in refs), dtype=np.int32, count=len(refs)),
            np.fromiter((r.block_id for r in refs), dtype=np.int64, count=len(refs)))


def _as_int64(query, out: np.ndarray) -> int:
    n = len(query)
    if n > out.shape[0]:
        raise ValueError(f"query of {n} tokens exceeds pool staging ({out.shape[0]})")
    if n:
        if isinstance(query, np.ndarray):
            out[:n] = query
        else:
            out[:n] = np.fromiter(query, dtype=np.int64, count=n)
    return n


class BlockPool:
    """One worker's KV pool (kvstore.py:59-250), on the GPU.

    capacity_blocks / block_size as in the reference. `records` is the
    initial number of record slots (grown on demand unless `kv_pages` fixes
    it: a KV-backed pool maps record slot == physical KV page).
    """

    CapacityError: type = CapacityExhausted
    UNDERFLOW_ERROR: type = RuntimeError
    DEFAULT_MAX_QUERY = 1 << 17

    def __init__(self, capacity_blocks: int, block_size: int, *, device: int = 0,
                 records: int | None = None, kv_pages: int | None = None,
                 max_query_tokens: int | None = None, stream: int = 0) -> None:
        if capacity_blocks < 0 or block_size < 1:  # kvstore.py:64-65
            raise ValueError("capacity_blocks >= 0 and block_size >= 1 required")
        self.capacity_blocks = capacity_blocks
        self.block_size = block_size
        self.device = device
        self.stream = stream
        self._fixed = kv_pages is not None
        if kv_pages is not None:
            if capacity_blocks > kv_pages:
                raise ValueError("capacity_blocks exceeds the KV pages backing the pool")
            recs = kv_pages
        else:
            recs = records or max(1, min(capacity_blocks, 4096))
        mq = max_query_tokens or self.DEFAULT_MAX_QUERY
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.psk_pool_create(C.byref(h), capacity_blocks, block_size, recs, mq, device))
        self._h = h
        self._lib = lib
        ptrs = [C.c_void_p() for _ in range(6)]
        _lib.check(lib.psk_pool_host_buffers(h, *[C.byref(p) for p in ptrs]))
        self._tok = np.ctypeslib.as_array(C.cast(ptrs[0], C.POINTER(C.c_int64)), shape=(mq,))
        self._in_slots = np.ctypeslib.as_array(C.cast(ptrs[1], C.POINTER(C.c_int32)), shape=(mq,))
        self._in_ids = np.ctypeslib.as_array(C.cast(ptrs[2], C.POINTER(C.c_int64)), shape=(mq,))
        self._out_slots = np.ctypeslib.as_array(C.cast(ptrs[3], C.POINTER(C.c_int32)), shape=(mq,))
        self._out_ids = np.ctypeslib.as_array(C.cast(ptrs[4], C.POINTER(C.c_int64)), shape=(mq,))
        self._res = _lib.PoolResult.from_address(ptrs[5].value)
        self._max_q = mq
        self._ns_ids: dict[str, int] = {}
        self._ns_names: list[str] = []
        self._ns_inserted: list[str] = []  # order of first footprint entry
        self._staged = None  # last staged token object (identity cache)
        self._used = 0
        self.matched_tokens = 0
        self.lookup_tokens = 0
        self.eviction_count = 0
        self._next_block_id = 0

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.psk_pool_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- internals -------------------------------------------------------

    def _ns_id(self, ns: str) -> int:
        i = self._ns_ids.get(ns)
        if i is None:
            i = len(self._ns_names)
            if i >= 1024:
                raise ValueError("too many namespaces (max 1024)")
            self._ns_ids[ns] = i
            self._ns_names.append(ns)
        return i

    def _ns_name(self, i: int) -> str:
        return self._ns_names[int(i)]

    def _stage(self, query) -> int:
        if query is self._staged:
            return len(query)
        n = _as_int64(query, self._tok)
        self._staged = query if isinstance(query, tuple) else None
        return n

    def _absorb(self) -> None:
        r = self._res
        self._used = r.used_blocks
        self.matched_tokens = r.matched_tokens
        self.lookup_tokens = r.lookup_tokens
        self.eviction_count = r.eviction_count
        self._next_block_id = r.next_block_id

    def _ensure_records(self, n_full: int) -> None:
        if self._fixed:
            return
        need = min(self.capacity_blocks, self._used + n_full)
        have = _lib.load().psk_pool_records(self._h)
        if need > have:
            _lib.check(self._lib.psk_pool_reserve(self._h, max(need, 2 * have)))

    def _read_record(self, slot: int, block_id: int):
        fields = (C.c_int64 * 7)()
        toks = np.empty(self.block_size, dtype=np.int64)
        _lib.check(self._lib.psk_pool_read_record(self._h, slot, fields,
                                                  toks.ctypes.data_as(C.c_void_p)))
        if fields[0] != block_id:
            raise RuntimeError(f"block {block_id} is no longer resident (slot {slot} reused)")
        return list(fields), tuple(int(t) for t in toks)

    # -- queries ---------------------------------------------------------

    @property
    def used_blocks(self) -> int:
        return self._used

    @property
    def free_blocks(self) -> int:
        return self.capacity_blocks - self._used

    def stats(self) -> PoolStats:
        return PoolStats(
            capacity_blocks=self.capacity_blocks,
            used_blocks=self.used_blocks,
            free_blocks=self.free_blocks,
            matched_tokens=self.matched_tokens,
            lookup_tokens=self.lookup_tokens,
            eviction_count=self.eviction_count,
        )

    def _footprints(self) -> tuple[dict[str, int], dict[str, int]]:
        fp: dict[str, int] = {}
        pk: dict[str, int] = {}
        for ns in self._ns_inserted:
            a, b = C.c_int64(), C.c_int64()
            _lib.check(self._lib.psk_pool_footprint(self._h, self._ns_ids[ns], C.byref(a), C.byref(b)))
            fp[ns], pk[ns] = a.value, b.value
        return fp, pk

    def footprint_tokens(self) -> dict[str, int]:
        return self._footprints()[0]

    def peak_footprint_tokens(self) -> dict[str, int]:
        return self._footprints()[1]

    # -- operations ------------------------------------------------------

    def _walk(self, ns: str, query) -> BlockChain:
        n = self._stage(query)
        _lib.check(self._lib.psk_pool_lookup(self._h, self._ns_id(ns), None, n, 0, 0, self.stream))
        m = self._res.count
        return BlockChain(self, self._out_slots[:m].copy(), self._out_ids[:m].copy())

    def longest_prefix_match(self, ns: str, query, now: int) -> tuple[int, BlockChain]:
        """kvstore.py:123-138: pins the matched chain; caller must release()."""
        n = self._stage(query)
        _lib.check(self._lib.psk_pool_lookup(self._h, self._ns_id(ns), None, n, now, 1, self.stream))
        self._absorb()
        m = self._res.count
        chain = BlockChain(self, self._out_slots[:m].copy(), self._out_ids[:m].copy())
        return m * self.block_size, chain

    def insert(self, ns: str, seq, now: int) -> BlockChain:
        """kvstore.py:140-189: cache all full blocks of seq; new blocks are
        returned unpinned. Raises CapacityExhausted (partial evictions kept)."""
        n = self._stage(seq)
        self._ensure_records(n // self.block_size)
        code = self._lib.psk_pool_insert(self._h, self._ns_id(ns), None, n, now, self.stream)
        if code not in (_lib.PSK_OK, _lib.PSK_ECAPACITY, _lib.PSK_ECAPACITY_NEED):
            _lib.check(code)
        self._absorb()
        if code in (_lib.PSK_ECAPACITY_NEED, _lib.PSK_ECAPACITY):
            need = n // self.block_size - len(self._walk(ns, seq))  # kvstore.py:150
            if code == _lib.PSK_ECAPACITY_NEED:
                raise self.CapacityError(
                    f"need {need} blocks exceeds capacity {self.capacity_blocks}")
            raise self.CapacityError(f"cannot free {need} blocks: all remaining blocks pinned")
        m = self._res.count
        if m and ns not in self._ns_inserted:
            self._ns_inserted.append(ns)
        return BlockChain(self, self._out_slots[:m].copy(), self._out_ids[:m].copy())

    def evict_until(self, need: int) -> int:
        """kvstore.py:191-210."""
        code = self._lib.psk_pool_evict_until(self._h, need, self.stream)
        if code == _lib.PSK_ECAPACITY_NEED:
            raise self.CapacityError(f"need {need} blocks exceeds capacity {self.capacity_blocks}")
        if code not in (_lib.PSK_OK, _lib.PSK_ECAPACITY):
            _lib.check(code)
        self._absorb()
        if code == _lib.PSK_ECAPACITY:
            raise self.CapacityError(f"cannot free {need} blocks: all remaining blocks pinned")
        return int(self._res.evicted)

    def _stage_handles(self, blocks) -> int:
        s, b = _handles_of(blocks)
        n = len(b)
        if n > self._max_q:
            raise ValueError("too many block handles for one call")
        self._in_slots[:n] = s
        self._in_ids[:n] = b
        return n

    @property
    def max_handles(self) -> int:
        """Block handles one pin / release call takes."""
        return self._max_q

    def pin(self, blocks, now: int) -> None:
        """kvstore.py:237-240."""
        n = self._stage_handles(blocks)
        code = self._lib.psk_pool_pin(self._h, n, now, self.stream)
        if code == _lib.PSK_EINVAL:
            raise RuntimeError(_lib.last_error() or f"pin of a non-resident block {self._res.err_block_id}")
        _lib.check(code)

    def release(self, blocks) -> None:
        """kvstore.py:242-250: underflow raises RuntimeError after releasing
        the blocks that precede the offending one."""
        n = self._stage_handles(blocks)
        code = self._lib.psk_pool_release(self._h, n, self.stream)
        if code in (_lib.PSK_EUNDERFLOW, _lib.PSK_EINVAL):
            raise self.UNDERFLOW_ERROR(f"release underflow on block {self._res.err_block_id}")
        _lib.check(code)

    # -- debugging -------------------------------------------------------

    def _snapshot(self):
        R = int(self._lib.psk_pool_records(self._h))
        bid = np.empty(R, np.int64)
        par = np.empty(R, np.int64)
        ns = np.empty(R, np.int32)
        ref = np.empty(R, np.int32)
        ch = np.empty(R, np.int32)
        last = np.empty(R, np.int64)
        tok = np.empty(R * self.block_size, np.int64)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _lib.check(self._lib.psk_pool_snapshot(self._h, p(bid), p(par), p(ns), p(ref), p(ch),
                                               p(last), p(tok)))
        return bid, par, ns, ref, ch, last, tok.reshape(R, self.block_size)

    @property
    def _blocks(self) -> dict[int, KVBlock]:
        bid, par, ns, ref, ch, last, tok = self._snapshot()
        out: dict[int, KVBlock] = {}
        for s in np.nonzero(bid >= 0)[0].tolist():
            out[int(bid[s])] = KVBlock(
                block_id=int(bid[s]), namespace=self._ns_name(ns[s]),
                token_span=tuple(int(t) for t in tok[s]), ref_count=int(ref[s]),
                last_access=int(last[s]), parent_id=int(par[s]), child_count=int(ch[s]))
        return dict(sorted(out.items()))

    def dump_tree(self) -> str:
        """Same text format as kvstore.py:254-281."""
        blocks = self._blocks
        kids: dict[tuple[str, int], list[KVBlock]] = {}
        for b in blocks.values():
            kids.setdefault((b.namespace, b.parent_id), []).append(b)
        lines: list[str] = []

        def visit(ns: str, parent: int, path: tuple) -> None:
            for b in sorted(kids.get((ns, parent), []), key=lambda x: x.block_id):
                full = path + b.token_span
                digest = hashlib.sha1(",".join(map(str, full)).encode()).hexdigest()[:12]
                lines.append(f"{ns} {digest} {b.block_id} {b.ref_count} {b.last_access}")
                visit(ns, b.block_id, full)

        for ns in sorted({b.namespace for b in blocks.values()}):
            visit(ns, -1, ())
        return "\n".join(lines)
