"""Breakdown of the K7 pool API latency at the bench's 4096-token lookup
(bench.pool_ops): the Python drop-in calls vs the bare C-ABI calls vs an
empty launch + stream sync, wall clock per call (median of 200).

    python tools/pool_latency.py
"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_12029_b200 import _lib  # noqa: E402
from paper_2602_12029_b200.kvstore import BlockPool  # noqa: E402


def med(fn, n=200):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e6, 1)


pool = BlockPool(8192, 16)
q = tuple((7 << 32) | i for i in range(4096))
pool.insert("shared", q, 1)
lib = _lib.load()
ns = pool._ns_id("shared")
n = pool._stage(q)


def py_match_release():
    _, ch = pool.longest_prefix_match("shared", q, 2)
    pool.release(ch)


def c_lookup():
    lib.psk_pool_lookup(pool._h, ns, None, n, 0, 0, pool.stream)


def c_lookup_pin():
    lib.psk_pool_lookup(pool._h, ns, None, n, 3, 1, pool.stream)


s = torch.cuda.Stream()
x = torch.zeros(1, device="cuda")


def empty_launch_sync():
    x.add_(1)
    torch.cuda.synchronize()


print({"py_longest_prefix_match+release_us": med(py_match_release),
       "c_lookup_us": med(c_lookup),
       "torch_launch+sync_us": med(empty_launch_sync)})
