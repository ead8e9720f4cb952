"""Run the multi-model agent workload (BASELINE configs 3/5 semantics) on one
GPU in both serving modes and print req/s, p95 E2E, prefill tokens and the
prefix hit ratio; one JSON line per (rate, cap) point, so lists sweep the
reference's arrival-rate (A4) and concurrency-cap (A3) axes on the real
engine. --out DIR writes, per point and mode, the
reference's output files: workload.json, report.json, requests.csv, trace.txt
(schemas of metrics.py:17-91 / workload.py:159-195).

    python tools/run_agents.py [--shape 8b|tiny] [--rate 8[,4,...]] [--cap 0[,40,...]]
                               [--duration 20] [--pattern react] [--rows 64] [--out DIR]
    python tools/run_agents.py --sweep arrival_rate --values 2,4,8 --auto-concurrency [--out DIR]
        (the reference's sweep protocol, experiment.py: per-cell seeds,
        best cap of DEFAULT_CAP_GRID per cell, sweep.csv)
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2602_12029_b200 import workload as wl  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights  # noqa: E402
from paper_2602_12029_b200.router import ServingMode  # noqa: E402
from paper_2602_12029_b200.serve import (AgentServer, build_report, records_to_csv,  # noqa: E402
                                         report_to_json, summarize)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="8b")
    ap.add_argument("--rate", default="8", help="arrival rate(s), comma-separated")
    ap.add_argument("--cap", default="0", help="max concurrent sessions (0 = unbounded), comma-separated")
    ap.add_argument("--out", default=None, help="directory for workload.json / report.json / requests.csv")
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--pattern", default="react")
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--time-scale", type=float, default=1.0)
    ap.add_argument("--pool-pages", type=int, default=7500)
    ap.add_argument("--no-batch", action="store_true", help="one prefill forward per request (FCFS)")
    ap.add_argument("--modes", default="baseline,prefillshare")
    ap.add_argument("--host-tier-blocks", type=int, default=0, help="host staging tier behind the prefix pool")
    ap.add_argument("--max-context", type=int, default=None,
                    help="longest context (default: 4096 for react, 5120 for reflexion: 512 + 12 x (96 + 256))")
    ap.add_argument("--sweep", default=None, choices=["arrival_rate", "max_concurrent_sessions"],
                    help="the reference's sweep protocol (experiment.py): one axis, per-cell seeds, sweep.csv")
    ap.add_argument("--values", default=None, help="sweep axis values, comma-separated")
    ap.add_argument("--auto-concurrency", action="store_true",
                    help="arrival_rate sweeps: best cap of DEFAULT_CAP_GRID per cell (throughput)")
    ap.add_argument("--cap-grid", default=None, help="override DEFAULT_CAP_GRID, comma-separated")
    ap.add_argument("--initial-prompt-len", type=int, default=None)
    ap.add_argument("--merged-pool", action="store_true", help="PREFILLSHARE: one merged pool (not the fleet's)")
    ap.add_argument("--turns", type=int, default=None)
    ap.add_argument("--handoff", default="pin", choices=["pin", "copy"],
                    help="copy: decode-side residency budget + staged handoff (the reference fleet)")
    ap.add_argument("--decode-capacity", type=int, default=4500, help="decode budget per model, blocks")
    a = ap.parse_args()
    max_ctx = a.max_context or (5120 if a.pattern == "reflexion" else 4096)
    cfg = (LlamaConfig.llama8b(max_pos=max_ctx + 512) if a.shape == "8b"
           else LlamaConfig.tiny(max_pos=max_ctx + 512))
    models = list(wl.DEFAULT_MODELS)
    mods = [ModuleWeights(cfg, 100 + i) for i in range(len(models))]
    base = ModuleWeights(cfg, 99, with_head=False)
    if a.sweep:
        return run_sweep(a, cfg, models, mods, base, max_ctx)
    for rate in (float(x) for x in a.rate.split(",")):
        for cap in (int(x) for x in a.cap.split(",")):
            sessions = wl.generate(wl.WorkloadConfig(pattern=a.pattern, arrival_rate_per_s=rate,
                                                     duration_s=a.duration, seed=a.seed))
            out = {"workload": {"pattern": a.pattern, "rate": rate, "duration_s": a.duration, "cap": cap,
                                "sessions": len(sessions), "requests": sum(s.total_requests for s in sessions)},
                   "shape": a.shape, "prefill_batch": not a.no_batch, "rows_per_model": a.rows}
            point = None
            if a.out:
                point = Path(a.out) / f"{a.pattern}_rate{rate:g}_cap{cap}"
                point.mkdir(parents=True, exist_ok=True)
                (point / "workload.json").write_text(wl.export_sessions(sessions))
            for mode in (ServingMode(m) for m in a.modes.split(",")):
                srv = AgentServer(cfg, models, mode, rows_per_module=a.rows, pool_pages_per_worker=a.pool_pages,
                                  max_context=max_ctx, max_output=256, modules=mods, base=base,
                                  prefill_batch=not a.no_batch, host_tier_blocks=a.host_tier_blocks,
                                  merged_pool=a.merged_pool)
                recs = srv.run(sessions, max_concurrent=cap or None, time_scale=a.time_scale,
                               record_trace=point is not None)
                out[mode.value] = summarize(recs)
                out[mode.value]["gpu_time"] = srv.gpu_time()
                if srv.tier is not None:
                    out[mode.value]["host_tier"] = srv.tier.stats()
                if point is not None:
                    echo = {"mode": mode.value, "workload": out["workload"], "shape": a.shape,
                            "rows_per_model": a.rows, "pool_blocks_per_worker": a.pool_pages}
                    (point / f"report_{mode.value}.json").write_text(report_to_json(build_report(srv, recs, echo)))
                    (point / f"requests_{mode.value}.csv").write_text(records_to_csv(recs))
                    (point / f"trace_{mode.value}.txt").write_text("\n".join(srv.trace) + "\n")
                del srv
                torch.cuda.empty_cache()
            b, p = out.get("baseline", {}), out.get("prefillshare", {})
            if b.get("req_per_s") and p.get("req_per_s"):
                out["throughput_ratio"] = p["req_per_s"] / b["req_per_s"]
                out["p95_ratio"] = b["p95_e2e_ms"] / p["p95_e2e_ms"]
            print(json.dumps(out), flush=True)


def run_sweep(a, cfg, models, mods, base, max_ctx):
    """the reference's sweep protocol on the real engine."""
    from paper_2602_12029_b200 import sweep
    out = Path(a.out) if a.out else None
    if out:
        out.mkdir(parents=True, exist_ok=True)

    def run(sessions, mode, cap):
        srv = AgentServer(cfg, models, ServingMode(mode), rows_per_module=a.rows, pool_pages_per_worker=a.pool_pages,
                          max_context=max_ctx, max_output=256, modules=mods, base=base,
                          prefill_batch=not a.no_batch, merged_pool=a.merged_pool, handoff=a.handoff,
                          decode_capacity_blocks=a.decode_capacity)
        recs = srv.run(sessions, max_concurrent=cap or None, time_scale=a.time_scale)
        echo = {"mode": mode, "cap": cap, "shape": a.shape, "rows_per_model": a.rows,
                "pool_blocks_per_worker": a.pool_pages, "sessions": len(sessions)}
        rep = build_report(srv, recs, echo)
        rep["summary"] = summarize(recs)
        rep["gpu_time"] = srv.gpu_time()
        line = {"mode": mode, "cap": cap, **{k: rep[k] for k in ("throughput_tok_per_s", "p95_e2e_us", "mean_ttft_us",
                                                                  "prefix_hit_ratio", "eviction_count",
                                                                  "failure_count")},
                "req_per_s": rep["summary"].get("req_per_s"), "staging_handoff_count": rep["staging_handoff_count"],
                "p95_ttft_us": rep["p95_ttft_us"], "completed": rep["completed_count"]}
        print(json.dumps(line), flush=True)
        del srv
        torch.cuda.empty_cache()
        return rep

    base_wl = wl.WorkloadConfig(pattern=a.pattern, arrival_rate_per_s=float(a.rate.split(",")[0]),
                                duration_s=a.duration, initial_prompt_len=a.initial_prompt_len, turns=a.turns)
    grid = tuple(int(x) for x in a.cap_grid.split(",")) if a.cap_grid else sweep.DEFAULT_CAP_GRID
    values = [float(x) if a.sweep == "arrival_rate" else int(x) for x in a.values.split(",")]
    cells = sweep.run_sweep(run, base_wl, a.seed, a.sweep, values, a.modes.split(","),
                            auto_concurrency=a.auto_concurrency, cap_grid=grid,
                            default_cap=int(a.cap.split(",")[0]))
    table = sweep.sweep_table(cells)
    print(table, flush=True)
    if out:
        (out / "sweep.csv").write_text(table)
        (out / "cells.jsonl").write_text("".join(json.dumps({"axis": c.axis, "value": c.value, "mode": c.mode,
                                                             "cap": c.cap, "chosen_cap": c.chosen_cap,
                                                             "report": c.report}) + "\n" for c in cells))


if __name__ == "__main__":
    main()
