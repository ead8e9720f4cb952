"""Agent-workload serving loop (serve.py): metric definitions on CPU
(metrics.py:22-42 semantics) and, on the GPU, a short tiny-model workload in
both serving modes: every request completes, and PrefillShare prefills fewer
tokens with a higher prefix-hit ratio than the per-model baseline (the
reference's A1/A3 direction, test_acceptance.py:37-147)."""

import pytest

from paper_2602_12029_b200.serve import RequestRecord, summarize


def test_summarize_nearest_rank_and_window():
    recs = []
    for i in range(20):
        r = RequestRecord(i, 0, "m", issue_us=i * 1e5)
        r.first_token_us = r.issue_us + 1e4
        r.done_us = r.issue_us + (i + 1) * 1e5
        r.out_tokens = 10
        recs.append(r)
    s = summarize(recs, warmup_fraction=0.1)
    e2e = sorted((i + 1) * 1e5 for i in range(20))
    assert s["p95_e2e_ms"] == e2e[18] / 1e3  # ceil(0.95*20) - 1 = 18
    t_end = max(r.done_us for r in recs)
    win = [r for r in recs if r.done_us >= 0.1 * t_end]
    assert abs(s["req_per_s"] - len(win) / (0.9 * t_end / 1e6)) < 1e-9
    assert summarize([]) == {"completed": 0, "failed": 0}


@pytest.mark.gpu
@pytest.mark.parametrize("rows,batch", [(4, False), (4, True), (12, True)])
def test_agent_workload_tiny_both_modes(rows, batch):
    """Both serving modes through the real engine: FCFS one-forward-per-request
    prefills and batched partial prefills; 12 rows per module runs the decode
    GEMVs on K5-TC."""
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights
    from paper_2602_12029_b200.router import ServingMode
    from paper_2602_12029_b200.serve import AgentServer
    cfg = LlamaConfig.tiny(max_pos=4096)
    models = list(wl.DEFAULT_MODELS)
    sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=3.0, duration_s=2.0,
                                             seed=1, turns=2))
    n_req = sum(s.total_requests for s in sessions)
    mods = [ModuleWeights(cfg, 10 + i) for i in range(4)]
    base = ModuleWeights(cfg, 9, with_head=False)
    res = {}
    for mode in (ServingMode.BASELINE, ServingMode.PREFILLSHARE):
        srv = AgentServer(cfg, models, mode, rows_per_module=rows, pool_pages_per_worker=512,
                          max_context=4096, max_output=128, modules=mods, base=base, prefill_batch=batch)
        recs = srv.run(sessions)
        assert len(recs) == n_req and all(r.done_us is not None for r in recs)
        assert all(r.out_tokens == 128 for r in recs)
        res[mode] = summarize(recs)
        gt = srv.gpu_time()
        assert gt["decode_steps"] > 0 and gt["prefill_calls"] > 0
    b, p = res[ServingMode.BASELINE], res[ServingMode.PREFILLSHARE]
    assert p["prefill_tokens"] < b["prefill_tokens"]
    assert p["prefix_hit_ratio"] > b["prefix_hit_ratio"]
