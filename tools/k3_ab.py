"""K3 A/B: variants of the prefill attention kernel given as
name:KEY=VAL;KEY=VAL (env of the child; e.g. PSK_PREFILL_SPLIT=1, or
PSK_LIB=<variant .so>), alternating child processes (variants are read once
per process), min / median of per-child timings of the 4k causal attention
(32 layers cycled, CUDA-graph replay, SM clock sampled while timing).

    python tools/k3_ab.py [reps] [T]
"""
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
T = sys.argv[2] if len(sys.argv) > 2 else "4096"
# extra args: name:KEY=VAL;KEY=VAL variants (default: TMEM-P vs shared-memory-P)
variants = [("tmem-P", {}), ("smem-P", {"PSK_PREFILL_PSMEM": "1"})]
if len(sys.argv) > 3:
    variants = []
    for a in sys.argv[3:]:
        name, _, kv = a.partition(":")
        variants.append((name, dict(x.split("=", 1) for x in kv.split(";") if x)))
res = {name: [] for name, _ in variants}
for rep in range(reps):
    for name, env in variants:
        r = subprocess.run([sys.executable, str(ROOT / "tools" / "bench_prefill.py"), T, "attnonly"],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        for line in r.stdout.splitlines():
            if line.startswith("prefill attention"):
                us = float(line.split(":")[1].split("us")[0])
                clk = int(line.split("sm_clock_median=")[1].split()[0]) if "sm_clock_median=" in line else -1
                res[name].append((us, clk))
                print(f"{name} rep{rep}: {line}", flush=True)
        if r.returncode:
            print(r.stderr[-2000:])
for name, v in res.items():
    if v:
        us = [x[0] for x in v]
        # cycles per layer (us x MHz) removes the power-cap clock drift between runs
        cyc = [x[0] * x[1] for x in v if x[1] > 0]
        print(f"{name}: median {statistics.median(us):.1f} us/layer, min {min(us):.1f} (n={len(us)}); "
              f"median {statistics.median(cyc) / 1e3 if cyc else -1:.1f} kcycles/layer")
