"""The reference's discrete-event simulator (virtual time, its cost model)
on the exact workload trace our real engine served, both modes, next to the
engine's report (the reference DES shown beside the real
engine's req/s and p95). Runs where /root/reference is importable (this
container, not the GPU box); writes one JSON object.

    python tools/ref_des.py profiles/r01_agents_runs/react_rate8_cap0 > profiles/r01_ref_des_rate8.json
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from prefillsim import workload as rwl  # noqa: E402
from prefillsim.config import RunSettings, SimConfig  # noqa: E402
from prefillsim.experiment import run_once  # noqa: E402

KEYS = ("request_count", "completed_count", "failure_count", "p95_e2e_us", "p95_ttft_us", "mean_ttft_us",
        "throughput_tok_per_s", "prefix_hit_ratio", "end_time_us")

point = Path(sys.argv[1])
sessions = rwl.import_sessions((point / "workload.json").read_text())
out = {"workload": str(point / "workload.json"), "sessions": len(sessions), "modes": {}}
for mode in ("baseline", "prefillshare"):
    cfg = SimConfig(run=RunSettings(mode=mode, seed=0))
    _, rep = run_once(cfg, sessions=sessions)
    eng = json.loads((point / f"report_{mode}.json").read_text())
    out["modes"][mode] = {"reference_des": {k: rep[k] for k in KEYS},
                          "engine_b200": {k: eng.get(k) for k in KEYS}}
for side in ("reference_des", "engine_b200"):
    b = out["modes"]["baseline"][side]
    p = out["modes"]["prefillshare"][side]
    out[side + "_ratios"] = {"throughput": p["throughput_tok_per_s"] / b["throughput_tok_per_s"],
                             "p95_e2e": b["p95_e2e_us"] / p["p95_e2e_us"]}
print(json.dumps(out, indent=1))
