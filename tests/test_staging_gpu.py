"""Host staging tier behind the prefix pool (staging.py):
write-through copies of computed blocks, bit-exact H2D reload into new
pages, and the agent server recomputing less when the GPU pool evicts."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_tier_roundtrip_bit_exact():
    from paper_2602_12029_b200.model import KVCache, LlamaConfig, ModuleWeights, PrefillRunner
    from paper_2602_12029_b200.staging import HostKVTier, block_edges, block_keys
    cfg = LlamaConfig.tiny()
    base = ModuleWeights(cfg, 1, with_head=False)
    kv = KVCache(cfg, 40)
    pre = PrefillRunner(cfg, base, kv, max_tokens=512)
    rng = np.random.default_rng(0)
    ctx = rng.integers(0, cfg.vocab, 300)
    pages = list(range(3, 3 + 19))
    pre.run(torch.from_numpy(ctx).cuda(), 0, torch.tensor(pages, dtype=torch.int32, device="cuda"))
    tier = HostKVTier(kv, capacity_blocks=8)
    keys = block_keys("shared", ctx, 18)
    ed = block_edges("shared", ctx, keys, 0, 18)
    tier.store(keys[:6], ed[:6], pages[:6])
    tier.store(keys[6:14], ed[6:14], pages[6:14])  # LRU: the first 6 are evicted from the 8-block tier
    want = kv.data[pages[6:14]].clone()
    assert tier.lookup(keys[:6], ed[:6]) == []
    slots = tier.lookup(keys[6:14], ed[6:14])
    assert len(slots) == 8
    new_pages = list(range(25, 33))
    kv.data[new_pages].zero_()
    tier.reload(slots, new_pages)
    torch.cuda.synchronize()
    assert torch.equal(kv.data[new_pages], want)
    assert block_keys("shared", ctx, 3) == keys[:3] and block_keys("model:a", ctx, 1) != keys[:1]
    assert tier.stats()["reloaded"] == 8


def test_agent_server_reloads_evicted_prefix_blocks():
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights
    from paper_2602_12029_b200.router import ServingMode
    from paper_2602_12029_b200.serve import AgentServer, summarize
    cfg = LlamaConfig.tiny(max_pos=4096)
    models = list(wl.DEFAULT_MODELS)
    sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=6.0, duration_s=2.0, seed=3,
                                             turns=2))
    n_req = sum(s.total_requests for s in sessions)
    mods = [ModuleWeights(cfg, 10 + i) for i in range(4)]
    base = ModuleWeights(cfg, 9, with_head=False)
    res = {}
    for tier in (0, 4096):
        # a small merged shared pool (4 x 130 blocks, active sessions compete): later agents' prefixes get evicted
        srv = AgentServer(cfg, models, ServingMode.PREFILLSHARE, rows_per_module=1, pool_pages_per_worker=130,
                          max_context=2048, max_output=128, modules=mods, base=base, host_tier_blocks=tier,
                          merged_pool=True)
        recs = srv.run(sessions, time_scale=0.2)
        assert all(r.done_us is not None and not r.failed for r in recs) and len(recs) == n_req
        res[tier] = (summarize(recs), srv.tier.stats() if srv.tier else None, srv.pools[0].eviction_count)
    (s0, _, ev0), (s1, st1, ev1) = res[0], res[4096]
    assert ev0 > 0 and ev1 > 0, (res, n_req)            # the pool did evict
    assert st1["reloaded"] > 0 and st1["stored"] > 0
    # (the prefill-token totals of the two real-time runs are not comparable:
    # arrival timing changes the LRU order; the reload itself is checked bit
    # for bit in test_tier_roundtrip_bit_exact)


def test_decode_residency_stage_reload_bit_exact():
    """DecodeResidency: a context staged to pinned host memory and reloaded
    into other decode pages is bit-identical (the staged handoff moves the
    same bytes); the budget accounting follows take / give."""
    from paper_2602_12029_b200.model import KVCache, LlamaConfig
    from paper_2602_12029_b200.staging import DecodeResidency
    cfg = LlamaConfig.tiny()
    kv = KVCache(cfg, 64)
    kv.data.copy_(torch.randn(kv.data.shape, device="cuda").to(torch.bfloat16))
    res = DecodeResidency(kv, first=40, capacity=20, threshold=0.9)
    src = [3, 9, 17, 2, 30]
    want = kv.data[src].clone()
    host = res.stage(src)
    kv.data[src].zero_()  # the prefill pool reuses the pages after the handoff
    res.fence()
    kv.data[src] = 0
    assert res.staged_count == 1 and res.staged_bytes == want.numel() * 2
    pages = res.take(5)
    assert all(40 <= p < 60 for p in pages) and res.resident == 5 and not res.must_stage(15)
    res.reload(host, pages)
    torch.cuda.synchronize()
    assert torch.equal(kv.data[pages], want)
    res.take(14)
    assert res.must_stage(1) and res.fraction() > 0.9   # 19 / 20 resident: above the threshold
    res.give(pages)
    assert res.resident == 14 and not res.must_stage(5)


@pytest.mark.parametrize("capacity", [130, 4096])
def test_agent_server_copy_handoff_with_staging(capacity):
    """handoff="copy" (the reference fleet's decode-side residency): contexts
    move into each decode worker's own budget, prefill pins drop at handoff;
    with a small budget most handoffs stage through host memory and reload.
    Every request completes, the trace keeps the life-cycle order with the
    staged flag, and staging_handoff_count reports the staged handoffs."""
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights
    from paper_2602_12029_b200.router import ServingMode
    from paper_2602_12029_b200.serve import AgentServer, build_report
    from test_serve import check_trace
    cfg = LlamaConfig.tiny(max_pos=4096)
    models = list(wl.DEFAULT_MODELS)
    sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=4.0, duration_s=2.0, seed=5,
                                             turns=2))
    n_req = sum(s.total_requests for s in sessions)
    mods = [ModuleWeights(cfg, 10 + i) for i in range(4)]
    base = ModuleWeights(cfg, 9, with_head=False)
    srv = AgentServer(cfg, models, ServingMode.PREFILLSHARE, rows_per_module=4, pool_pages_per_worker=512,
                      max_context=2048, max_output=128, modules=mods, base=base, handoff="copy",
                      decode_capacity_blocks=capacity)
    # the small budget needs contexts resident together: arrivals compressed
    # harder there (how many overlap otherwise depends on the decode speed)
    recs = srv.run(sessions, time_scale=0.3 if capacity > 130 else 0.05, record_trace=True)
    assert len(recs) == n_req and all(r.done_us is not None and not r.failed for r in recs)
    check_trace(srv.trace, sessions, n_req, len(models))
    rep = build_report(srv, recs, {"capacity": capacity})
    staged = sum(1 for ln in srv.trace if " HandoffComplete " in ln and ln.endswith("staged=1"))
    assert rep["staging_handoff_count"] == staged
    if capacity == 130:
        assert staged > 0
    else:
        assert staged == 0
    assert all(r.resident == 0 for r in srv.residency)  # every context left its budget
