"""K8 handoff host logic: world_size-2 gloo on CPU (prefill rank -> decode
rank page transfer with header), the page allocator, and (GPU) the
same-process page-copy kernel."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2602_12029_b200.transfer import HandoffMeta, PageAllocator, recv_pages, send_pages
    g = torch.Generator().manual_seed(7)
    prefill_pool = torch.randn(12, 256, generator=g).to(torch.bfloat16)
    try:
        if rank == 0:
            nbytes = send_pages(prefill_pool, [5, 2, 9, 11], 1, HandoffMeta(17, 3, 60, 1234))
            send_pages(prefill_pool, [], 1, HandoffMeta(18, 3, 1, 5))
            q.put(("sent", nbytes))
        else:
            pool = torch.zeros(8, 256, dtype=torch.bfloat16)
            alloc = PageAllocator(2, 6)
            pages, meta = recv_pages(pool, 0, alloc.alloc)
            ok = all(torch.equal(pool[p], prefill_pool[s]) for p, s in zip(pages, [5, 2, 9, 11]))
            pages2, meta2 = recv_pages(pool, 0, alloc.alloc)
            q.put(("recv", ok, pages, (meta.request_id, meta.session_id, meta.shared_len,
                                       meta.first_token, meta.n_pages), pages2, meta2.n_pages))
    finally:
        dist.destroy_process_group()


def test_handoff_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = {}
    while not q.empty():
        item = q.get()
        res[item[0]] = item[1:]
    assert all(p.exitcode == 0 for p in ps)
    assert res["sent"][0] == 4 * 256 * 2
    ok, pages, meta, pages2, n2 = res["recv"]
    assert ok and pages == [2, 3, 4, 5]
    assert meta == (17, 3, 60, 1234, 4) and pages2 == [] and n2 == 0


def test_page_allocator():
    from paper_2602_12029_b200.transfer import PageAllocator
    a = PageAllocator(10, 4)
    assert a.alloc(2) == [10, 11]
    a.release([10, 11])
    assert a.alloc(4) == [10, 11, 12, 13]
    with pytest.raises(MemoryError):
        a.alloc(1)


@pytest.mark.gpu
def test_copy_pages_kernel():
    from paper_2602_12029_b200.transfer import copy_pages
    src = torch.randn(10, 65536, device="cuda").to(torch.bfloat16)
    dst = torch.zeros(6, 65536, dtype=torch.bfloat16, device="cuda")
    copy_pages(src, dst, [9, 0, 4], [1, 5, 0])
    torch.cuda.synchronize()
    assert torch.equal(dst[1], src[9]) and torch.equal(dst[5], src[0]) and torch.equal(dst[0], src[4])
    assert dst[2].abs().sum().item() == 0
