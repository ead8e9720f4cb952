"""Host-tier index (staging.TierIndex) on CPU: a 64-bit key collision must
never reload another path's KV. The tier finds candidates by a rolling key
of the block's token path and verifies the block's exact edge (namespace,
parent key, 16 tokens), the reference's edge key (kvstore.py:69-70)."""

import numpy as np


def _ctx(seed, n=64):
    return np.random.default_rng(seed).integers(0, 1 << 40, n, dtype=np.int64)


def test_verified_lookup_roundtrip_and_lru():
    from paper_2602_12029_b200.staging import TierIndex, block_edges, block_keys
    idx = TierIndex(capacity=3)
    ctx = _ctx(0)
    keys = block_keys("shared", ctx, 4)
    ed = block_edges("shared", ctx, keys, 0, 4)
    slots = [idx.place(k, e) for k, e in zip(keys[:3], ed[:3])]
    assert sorted(slots) == [0, 1, 2] and idx.place(keys[0], ed[0]) is None  # present: touched, not re-stored
    assert idx.lookup(keys, ed) == [slots[0], slots[1], slots[2]]          # stops at the absent 4th block
    idx.place(keys[3], ed[3])                                               # evicts the LRU entry (block 0)
    assert idx.lookup(keys, ed) == [] and idx.lookup(keys[1:], ed[1:]) == slots[1:] + [slots[0]]


def test_key_collision_is_rejected():
    """Two different contexts whose block keys collide (forced: the second
    context is looked up under the first one's keys): no slot is returned,
    neither at the first block (different tokens) nor deeper (same tokens,
    different parent), nor across namespaces."""
    from paper_2602_12029_b200.staging import TierIndex, block_edges, block_keys
    idx = TierIndex(capacity=16)
    a = _ctx(1)
    ka = block_keys("shared", a, 4)
    ea = block_edges("shared", a, ka, 0, 4)
    for k, e in zip(ka, ea):
        idx.place(k, e)
    # 1) different tokens in block 0 under A's keys
    b = a.copy()
    b[3] += 1
    kb = block_keys("shared", b, 4)
    assert idx.lookup(ka, block_edges("shared", b, kb, 0, 4)) == []
    # 2) same block-1 tokens, different block 0: a collision at block 1 only
    #    (key(B1) == key(A1)) is caught by the parent key
    c = a.copy()
    c[0] += 1
    kc = block_keys("shared", c, 4)
    forced = [kc[0]] + ka[1:]
    assert idx.lookup(forced[1:], block_edges("shared", c, forced, 1, 4)) == []
    # 3) another namespace under the same keys
    assert idx.lookup(ka, block_edges("model:a", a, ka, 0, 4)) == []
    assert idx.collisions == 3
    # the genuine path still reloads in full
    assert len(idx.lookup(ka, ea)) == 4
