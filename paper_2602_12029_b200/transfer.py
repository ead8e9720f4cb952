"""Prefill -> decode KV handoff across GPUs (K8), one process per GPU.

The reference models the handoff as bytes / bandwidth (costs.py:66-83) and
serializes it with decode steps on the decode worker (cluster.py:370-412):
the FULL context's KV moves to the model's decode worker, then the prefill
pins are released (blocks stay cached on the prefill side).

Here the copy unit is the KV page (all layers of 16 positions; 2 MiB at the
8B shape, one contiguous run), so a handoff is one grouped NCCL P2P of page
views — no pack / unpack pass through HBM — preceded by a small header. On
NVLink 5 / NVSwitch every prefill GPU reaches every decode GPU at full
bandwidth. Within one process (same GPU or peer-mapped pools) use
`copy_pages` (psk_kv_copy_pages) instead; on one GPU the handoff is a
zero-copy pin.

Works with any torch.distributed backend that has P2P (NCCL on GPUs; gloo on
CPU, which the multi-process tests use).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

from . import _lib

HEADER_WORDS = 8


@dataclass
class HandoffMeta:
    request_id: int
    session_id: int
    shared_len: int      # positions the decode module attends to (n - 1)
    first_token: int     # last prompt token, processed by the decode module
    n_pages: int = 0


def _header(meta: HandoffMeta, n_pages: int, device) -> torch.Tensor:
    h = torch.zeros(HEADER_WORDS, dtype=torch.int64, device=device)
    h[:5] = torch.tensor([n_pages, meta.request_id, meta.session_id, meta.shared_len, meta.first_token])
    return h


def send_pages(pool: torch.Tensor, pages: list[int], dst: int, meta: HandoffMeta,
               group=None) -> int:
    """Prefill side: ship `pages` of `pool` ([n_pages, page_elems]) to rank
    `dst`. Returns the bytes moved."""
    dist.send(_header(meta, len(pages), pool.device), dst, group=group)
    ops = [dist.P2POp(dist.isend, pool[p], dst, group=group) for p in pages]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return len(pages) * pool[0].numel() * pool.element_size()


def recv_pages(pool: torch.Tensor, src: int, alloc: Callable[[int], list[int]],
               group=None) -> tuple[list[int], HandoffMeta]:
    """Decode side: receive one handoff from `src` into pages obtained from
    `alloc(n)` of the local pool. Returns (local pages, meta)."""
    h = torch.zeros(HEADER_WORDS, dtype=torch.int64, device=pool.device)
    dist.recv(h, src, group=group)
    n, rid, sid, slen, first = (int(x) for x in h[:5].tolist())
    pages = alloc(n)
    ops = [dist.P2POp(dist.irecv, pool[p], src, group=group) for p in pages]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return pages, HandoffMeta(rid, sid, slen, first, n)


def copy_pages(src_pool: torch.Tensor, dst_pool: torch.Tensor, src_pages: list[int],
               dst_pages: list[int], stream=None) -> None:
    """Same-process page move on the GPU (psk_kv_copy_pages)."""
    if len(src_pages) != len(dst_pages):
        raise ValueError("page lists differ in length")
    dev = src_pool.device
    sp = torch.tensor(src_pages, dtype=torch.int32, device=dev)
    dp = torch.tensor(dst_pages, dtype=torch.int32, device=dev)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    _lib.call("psk_kv_copy_pages", src_pool.data_ptr(), dst_pool.data_ptr(), sp.data_ptr(), dp.data_ptr(),
              len(src_pages), src_pool[0].numel() * src_pool.element_size(), s)


class PageAllocator:
    """Free list over a range of page indices (decode-side private pages and
    received handoffs). LIFO, deterministic."""

    def __init__(self, first: int, count: int):
        self.free = list(range(first + count - 1, first - 1, -1))

    def alloc(self, n: int) -> list[int]:
        if n > len(self.free):
            raise MemoryError(f"KV pages exhausted: need {n}, have {len(self.free)}")
        out = [self.free.pop() for _ in range(n)]
        return out

    def release(self, pages: list[int]) -> None:
        self.free.extend(reversed(pages))
