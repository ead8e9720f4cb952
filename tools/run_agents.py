"""Run the multi-model agent workload (BASELINE configs 3/5 semantics) on one
GPU in both serving modes and print req/s, p95 E2E, prefill tokens and the
prefix hit ratio.

    python tools/run_agents.py [--shape 8b|tiny] [--rate 1.0] [--duration 10]
                               [--pattern react] [--rows 8] [--time-scale 1]
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
from paper_2602_12029_b200.serve import AgentServer, summarize  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="8b")
    ap.add_argument("--rate", type=float, default=1.0)
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--pattern", default="react")
    ap.add_argument("--rows", type=int, default=16)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--time-scale", type=float, default=1.0)
    ap.add_argument("--pool-pages", type=int, default=7500)
    ap.add_argument("--no-batch", action="store_true", help="one prefill forward per request (FCFS)")
    ap.add_argument("--modes", default="baseline,prefillshare")
    a = ap.parse_args()
    cfg = LlamaConfig.llama8b(max_pos=4096 + 512) if a.shape == "8b" else LlamaConfig.tiny(max_pos=4096)
    models = list(wl.DEFAULT_MODELS)
    sessions = wl.generate(wl.WorkloadConfig(pattern=a.pattern, arrival_rate_per_s=a.rate,
                                             duration_s=a.duration, seed=a.seed))
    mods = [ModuleWeights(cfg, 100 + i) for i in range(len(models))]
    base = ModuleWeights(cfg, 99, with_head=False)
    out = {"workload": {"pattern": a.pattern, "rate": a.rate, "duration_s": a.duration,
                        "sessions": len(sessions), "requests": sum(s.total_requests for s in sessions)},
           "shape": a.shape}
    out["prefill_batch"] = not a.no_batch
    for mode in (ServingMode(m) for m in a.modes.split(",")):
        srv = AgentServer(cfg, models, mode, rows_per_module=a.rows, pool_pages_per_worker=a.pool_pages,
                          max_context=4096, max_output=256, modules=mods, base=base,
                          prefill_batch=not a.no_batch)
        recs = srv.run(sessions, time_scale=a.time_scale)
        out[mode.value] = summarize(recs)
        out[mode.value]["gpu_time"] = srv.gpu_time()
        del srv
        torch.cuda.empty_cache()
    b, p = out.get("baseline", {}), out.get("prefillshare", {})
    if b.get("req_per_s") and p.get("req_per_s"):
        out["throughput_ratio"] = p["req_per_s"] / b["req_per_s"]
        out["p95_ratio"] = b["p95_e2e_ms"] / p["p95_e2e_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
