"""K7 block pool parity.

CPU: the oracle (oracle/pool.py) replays every reference-generated op stream
(tests/golden/pool_streams.json.gz, produced by prefillsim.kvstore.BlockPool)
with identical outcomes — this pins the oracle.
GPU: the drop-in GPU pool replays the same streams bit-exactly, mirrors the
reference's hand scenarios (test_kvstore.py:23-156), and is compared with the
oracle on large random / eviction-heavy op streams.
"""

import random

import pytest

from pool_replay import GpuAdapter, OracleAdapter, expand_tokens, load_des_logs, load_streams, replay


def _stream_ids():
    return [s["name"] for s in load_streams()]


@pytest.mark.parametrize("name", _stream_ids())
def test_oracle_matches_reference_streams(name):
    stream = next(s for s in load_streams() if s["name"] == name)
    replay(stream, OracleAdapter)


def test_golden_streams_cover_edge_cases():
    streams = load_streams()
    errs = {rec["error"] for s in streams for rec in s["expect"]}
    assert {"capacity", "underflow", None} <= errs
    evictions = sum(s["expect"][-1]["evictions"] for s in streams)
    assert evictions > 1000
    assert any(len(expand_tokens(op)) >= 4096 for s in streams for op in s["ops"]
               if op["op"] == "insert")


def _des_ids():
    return [s["name"] for s in load_des_logs()]


def test_des_call_logs_cover_the_seam():
    """The recorded reference runs exercise every seam op, heavy eviction and
    capacity failures, in both serving modes."""
    logs = load_des_logs()
    assert {s["name"].split("_")[3] for s in logs} == {"baseline", "prefillshare"}
    kinds = {op["op"] for s in logs for op in s["ops"]}
    assert kinds == {"lookup", "insert", "pin", "release"}
    assert any(len(op["refs"]) == 2 for s in logs for op in s["ops"] if op["op"] == "release")
    assert sum(s["expect"][-1]["evictions"] for s in logs) > 500_000
    assert sum(1 for s in logs for e in s["expect"] if e["error"] == "capacity") > 100


@pytest.mark.parametrize("name", [n for n in _des_ids() if "cap100_" in n or n.endswith("prefillshare_cap7500_w3")])
def test_oracle_matches_des_call_logs(name):
    """The oracle pool on the reference's recorded seam traffic (the small
    pools: the oracle's argmin-scan eviction is O(capacity) per eviction)."""
    stream = next(s for s in load_des_logs() if s["name"] == name)
    replay(stream, OracleAdapter, check_digest_every=25)


# ----------------------------------------------------------------- GPU ----

gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("name", _stream_ids())
def test_gpu_pool_matches_reference_streams(name):
    stream = next(s for s in load_streams() if s["name"] == name)
    every = 1 if len(stream["ops"]) < 400 else 25
    a = replay(stream, GpuAdapter, check_digest_every=every)
    assert a.p.dump_tree() == stream["dump_tree"]


def _pool(cap, bs):
    from paper_2602_12029_b200.kvstore import BlockPool
    return BlockPool(capacity_blocks=cap, block_size=bs)


@gpu
def test_gpu_hand_scenarios():
    """test_kvstore.py:23-156, against the GPU pool."""
    from paper_2602_12029_b200.kvstore import CapacityExhausted
    pool = _pool(100, 4)
    pool.insert("ns", tuple(range(10)), now=1)
    matched, blocks = pool.longest_prefix_match("ns", tuple(range(10)), now=2)
    assert matched == 8
    assert [b.token_span for b in blocks] == [tuple(range(4)), tuple(range(4, 8))]
    pool.release(blocks)
    assert _pool(100, 16).insert("ns", tuple(range(15)), now=1) == []
    pool = _pool(100, 4)
    pool.insert("a", tuple(range(8)), now=1)
    matched, blocks = pool.longest_prefix_match("b", tuple(range(8)), now=2)
    assert matched == 0 and blocks == []
    # shared prefix stored once
    pool = _pool(100, 4)
    common = tuple(range(8))
    pool.insert("ns", common + (100, 101, 102, 103), now=1)
    pool.insert("ns", common + (200, 201, 202, 203), now=2)
    assert pool.used_blocks == 4 and pool.footprint_tokens()["ns"] == 16
    # LRU
    pool = _pool(2, 4)
    pool.insert("ns", (1, 2, 3, 4), now=1)
    pool.insert("ns", (5, 6, 7, 8), now=2)
    pool.insert("ns", (9, 10, 11, 12), now=3)
    assert pool.eviction_count == 1
    assert pool.longest_prefix_match("ns", (1, 2, 3, 4), now=4)[0] == 0
    # pinned survive
    pool = _pool(2, 4)
    pool.insert("ns", (1, 2, 3, 4), now=1)
    pool.insert("ns", (5, 6, 7, 8), now=2)
    _, pin_a = pool.longest_prefix_match("ns", (1, 2, 3, 4), now=3)
    _, pin_b = pool.longest_prefix_match("ns", (5, 6, 7, 8), now=4)
    with pytest.raises(CapacityExhausted):
        pool.insert("ns", (9, 10, 11, 12), now=5)
    pool.release(pin_a)
    pool.insert("ns", (9, 10, 11, 12), now=6)
    assert pool.eviction_count == 1
    pool.release(pin_b)
    # interior not evictable
    pool = _pool(2, 4)
    pool.insert("ns", tuple(range(8)), now=1)
    with pytest.raises(CapacityExhausted):
        pool.insert("ns", tuple(range(100, 112)), now=2)
    pool.insert("ns", tuple(range(100, 108)), now=3)
    assert pool.eviction_count == 2
    # underflow
    pool = _pool(4, 4)
    blocks = pool.insert("ns", (1, 2, 3, 4), now=1)
    pool.pin(blocks, now=1)
    pool.release(blocks)
    with pytest.raises(RuntimeError):
        pool.release(blocks)
    # need beyond capacity: no eviction
    pool = _pool(2, 4)
    pool.insert("ns", (1, 2, 3, 4), now=1)
    with pytest.raises(CapacityExhausted):
        pool.insert("ns", tuple(range(100, 112)), now=2)
    assert pool.eviction_count == 0
    # extending a matched chain does not evict it
    pool = _pool(2, 4)
    pool.insert("ns", (1, 2, 3, 4), now=1)
    pool.insert("ns", (5, 6, 7, 8), now=2)
    pool.insert("ns", (1, 2, 3, 4, 9, 10, 11, 12), now=3)
    matched, blocks = pool.longest_prefix_match("ns", (1, 2, 3, 4, 9, 10, 11, 12), now=4)
    assert matched == 8
    pool.release(blocks)
    # peak footprint
    pool = _pool(2, 4)
    pool.insert("ns", tuple(range(8)), now=1)
    assert pool.peak_footprint_tokens()["ns"] == 8
    pool.insert("ns", tuple(range(100, 104)), now=2)
    assert pool.footprint_tokens()["ns"] == 8 and pool.peak_footprint_tokens()["ns"] == 8
    # hit ratio
    pool = _pool(100, 4)
    pool.insert("ns", tuple(range(8)), now=1)
    _, blocks = pool.longest_prefix_match("ns", tuple(range(10)), now=2)
    pool.release(blocks)
    st = pool.stats()
    assert (st.matched_tokens, st.lookup_tokens, st.hit_ratio) == (8, 10, 0.8)


def _random_ops(rng, n_ops, bs, vocab, max_len, n_ns=3):
    for now in range(1, n_ops + 1):
        ns = f"ns{rng.randrange(n_ns)}"
        base = rng.randrange(vocab)
        length = rng.randrange(0, max_len)
        yield now, ns, tuple(base * 100_000 + (t if rng.random() < 0.97 else 7) for t in range(length))


@gpu
@pytest.mark.parametrize("bs,cap", [(1, 40), (16, 64), (16, 2000), (4, 7)])
def test_gpu_pool_random_vs_oracle(bs, cap):
    """Long random streams (beyond the golden ones) incl. eviction pressure."""
    from oracle.pool import OraclePool, OracleCapacityExhausted
    from paper_2602_12029_b200.kvstore import BlockPool, CapacityExhausted
    rng = random.Random(bs * 1000 + cap)
    g = BlockPool(cap, bs)
    o = OraclePool(cap, bs)
    held = []
    for now, ns, q in _random_ops(rng, 1500, bs, 12, 40 * bs):
        if rng.random() < 0.45:
            m, chain = g.longest_prefix_match(ns, q, now)
            ids = o.lookup(ns, q, now)
            assert chain.ids.tolist() == ids and m == len(ids) * bs
            held.append((chain, ids))
        else:
            e1 = e2 = None
            try:
                new = g.insert(ns, q, now)
            except CapacityExhausted:
                e1 = True
            try:
                want = o.insert(ns, q, now)
            except OracleCapacityExhausted:
                e2 = True
            assert e1 == e2
            if e1 is None:
                assert new.ids.tolist() == want
                if rng.random() < 0.5:
                    g.pin(new, now)
                    o.pin(want, now)
                    held.append((new, want))
        while len(held) > rng.randrange(1, 6):
            c, ids = held.pop(0)
            g.release(c)
            o.release(ids)
        assert (g.used_blocks, g.eviction_count, g.matched_tokens, g.lookup_tokens) == \
               (o.used_blocks, o.eviction_count, o.matched_tokens, o.lookup_tokens)
    got = sorted((b.block_id, b.namespace, b.token_span, b.parent_id, b.ref_count, b.last_access,
                  b.child_count) for b in g._blocks.values())
    assert got == o.state()


@gpu
def test_gpu_pool_long_contexts_and_growth():
    """32k-token contexts (2048 blocks per op) with record-table growth."""
    from oracle.pool import OraclePool
    from paper_2602_12029_b200.kvstore import BlockPool
    g = BlockPool(1 << 62, 16, records=64)
    o = OraclePool(1 << 62, 16)
    for s in range(6):
        base = (s + 1) << 32
        q = tuple(base | i for i in range(32768 + 5))
        assert g.insert("shared", q, s).ids.tolist() == o.insert("shared", q, s)
        m, chain = g.longest_prefix_match("shared", q + (1, 2, 3), 100 + s)
        assert m == 32768 and chain.ids.tolist() == o.lookup("shared", q + (1, 2, 3), 100 + s)
        g.release(chain)
        o.release(chain.ids.tolist())
    assert g.used_blocks == o.used_blocks == 6 * 2048


@gpu
@pytest.mark.parametrize("name", _des_ids())
def test_gpu_pool_matches_des_call_logs(name):
    """The pool seam proven on the reference's own traffic: every BlockPool
    call prefillsim.cluster.Simulation made while serving
    configs/fast_react.toml (both modes; 7500-, 1500- and 100-block pools)
    replayed through the GPU pool. Every outcome (matched tokens, block ids,
    CapacityExhausted), every counter after every op, the full block state
    every 25 ops and at the end, footprints and dump_tree equal the
    reference's."""
    stream = next(s for s in load_des_logs() if s["name"] == name)
    a = replay(stream, GpuAdapter, check_digest_every=25)
    if "dump_tree" in stream:
        assert a.p.dump_tree() == stream["dump_tree"]
