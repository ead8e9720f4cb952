"""K3 A/B: the TMEM-P kernel (default) vs the shared-memory-P kernel
(PSK_PREFILL_PSMEM=1), alternating child processes (the variant is read
once per process), medians of per-child timings of the 4k causal attention
(32 layers cycled, CUDA-graph replay).

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
res = {"tmem-P": [], "smem-P": []}
for rep in range(reps):
    for name, env in (("tmem-P", {}), ("smem-P", {"PSK_PREFILL_PSMEM": "1"})):
        r = subprocess.run([sys.executable, str(ROOT / "tools" / "bench_prefill.py"), T, "attn"],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        for line in r.stdout.splitlines():
            if line.startswith("prefill attention"):
                us = float(line.split(":")[1].split("us")[0])
                res[name].append(us)
                print(f"{name} rep{rep}: {line}", flush=True)
        if r.returncode:
            print(r.stderr[-2000:])
for name, v in res.items():
    if v:
        print(f"{name}: median {statistics.median(v):.1f} us/layer, min {min(v):.1f}, max {max(v):.1f} (n={len(v)})")
