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


def test_trace_line_matches_reference_format():
    """Lines produced by the reference's SimEvent.trace_line (core.py:146-150)
    for the same events, trailing space of an empty detail included."""
    from paper_2602_12029_b200.serve import trace_line
    assert trace_line(0, 0, "SessionArrival", 3) == "0 0 SessionArrival 3 -1 -1 "
    assert trace_line(1250.7, 7, "PrefillComplete", 3, 5, 0, "matched=32 new=100") == \
        "1250 7 PrefillComplete 3 5 0 matched=32 new=100"
    assert trace_line(99, 8, "DecodeStep", worker=4, detail="batch=2") == "99 8 DecodeStep -1 -1 4 batch=2"


def check_trace(trace, sessions, n_req, n_models):
    """Engine trace invariants: (time, seq) ordered, one arrival / completion
    per session, the request lifecycle in order, decode workers M + model."""
    from paper_2602_12029_b200.serve import TRACE_KINDS
    rows = [ln.split(" ", 6) for ln in trace]
    assert [int(r[1]) for r in rows] == list(range(len(rows)))
    times = [int(r[0]) for r in rows]
    assert times == sorted(times)
    kinds = [r[2] for r in rows]
    assert set(kinds) <= set(TRACE_KINDS)
    assert kinds.count("SessionArrival") == len(sessions) == kinds.count("SessionComplete")
    assert kinds.count("PrefillStart") == n_req == kinds.count("RequestComplete")
    order = {}
    for i, r in enumerate(rows):
        if r[2] in ("PrefillStart", "PrefillComplete", "HandoffComplete", "RequestComplete"):
            order.setdefault(int(r[4]), []).append(r[2])
        if r[2] in ("DecodeStep", "RequestComplete"):
            assert n_models <= int(r[5]) < 2 * n_models
    assert all(v == ["PrefillStart", "PrefillComplete", "HandoffComplete", "RequestComplete"]
               for v in order.values())


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
        recs = srv.run(sessions, record_trace=True)
        assert len(recs) == n_req and all(r.done_us is not None for r in recs)
        check_trace(srv.trace, sessions, n_req, len(models))
        assert all(r.out_tokens == 128 for r in recs)
        res[mode] = summarize(recs)
        gt = srv.gpu_time()
        assert gt["decode_steps"] > 0 and gt["prefill_calls"] > 0
        from paper_2602_12029_b200.serve import build_report, records_to_csv
        rep = build_report(srv, recs, {"mode": mode.value})
        assert set(rep) == REPORT_KEYS and rep["completed_count"] == n_req and rep["failure_count"] == 0
        assert rep["throughput_tok_per_s"] > 0 and len(records_to_csv(recs).splitlines()) == n_req + 1
    b, p = res[ServingMode.BASELINE], res[ServingMode.PREFILLSHARE]
    assert p["prefill_tokens"] < b["prefill_tokens"]
    assert p["prefix_hit_ratio"] > b["prefix_hit_ratio"]


REPORT_KEYS = {"schema_version", "config", "metadata", "end_time_us", "request_count", "completed_count",
               "failure_count", "staging_handoff_count", "p95_e2e_us", "mean_ttft_us", "p95_ttft_us",
               "throughput_tok_per_s", "prefix_hit_ratio", "matched_tokens", "lookup_tokens",
               "eviction_count", "peak_footprint_tokens", "peak_footprint_total"}


def test_report_and_csv_follow_reference_schema():
    """report.json / requests.csv of a real-engine run use the reference's
    fields and definitions (metrics.py:17-94): nearest-rank p95, windowed
    token throughput over per-step completions, pool aggregates summed over
    workers (cluster.py:232-252)."""
    from types import SimpleNamespace as NS

    from paper_2602_12029_b200.serve import (CSV_HEADER, RequestRecord, build_report, records_to_csv,
                                             report_to_json)
    recs = [RequestRecord(i, i // 2, f"model_{'ab'[i % 2]}", 100.0 * i, 100.0 * i + 50 + i, 100.0 * i + 900 + 7 * i,
                          128, 16 * i, 40) for i in range(20)]
    recs.append(RequestRecord(20, 10, "model_a", 2000.0, failed=True))
    pools = [NS(matched_tokens=300, lookup_tokens=1000, eviction_count=2,
                peak_footprint_tokens=lambda: {"shared": 640}),
             NS(matched_tokens=100, lookup_tokens=1000, eviction_count=1,
                peak_footprint_tokens=lambda: {"shared": 160, "model:x": 32})]
    comps = [(100 * k, 3) for k in range(1, 40)]
    srv = NS(token_completions=comps, pools=pools)
    rep = build_report(srv, recs, {"mode": "prefillshare"})
    assert set(rep) == REPORT_KEYS and rep["schema_version"] == 1
    e2e = sorted(int(r.done_us - r.issue_us) for r in recs[:20])
    assert rep["p95_e2e_us"] == e2e[18]                      # ceil(0.95 * 20) - 1
    assert rep["completed_count"] == 20 and rep["failure_count"] == 1 and rep["request_count"] == 21
    end = rep["end_time_us"]
    assert end == max(comps[-1][0], int(max(r.done_us for r in recs[:20])))
    want_tok = sum(n for t, n in comps if t >= 0.1 * end) / ((end - 0.1 * end) / 1e6)
    assert abs(rep["throughput_tok_per_s"] - want_tok) < 1e-9
    assert rep["prefix_hit_ratio"] == 400 / 2000 and rep["eviction_count"] == 3
    assert rep["peak_footprint_tokens"] == {"model:x": 32, "shared": 800} and rep["peak_footprint_total"] == 832
    assert report_to_json(rep).startswith("{")
    csv = records_to_csv(recs).splitlines()
    assert csv[0] == CSV_HEADER and len(csv) == 22
    assert csv[1] == "0,0,model_a,50,900,128" and csv[-1] == "20,10,model_a,,,0"
