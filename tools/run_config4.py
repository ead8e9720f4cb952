"""BASELINE configs[3] end to end on ONE B200, as far as it fits: 8B-shape
modules at full depth, a 32768-token shared context per session, M decode
modules (16 x 16 GB of weights need two GPUs; 8 fit next to the base
module), 256 greedy tokens per module. One PrefillShareEngine.serve per
batch: pool lookup / insert, the 32k shared prefill (kv_only), then every
module decodes from the shared pages (K6 reads each shared page once per
step for all M modules x 4 GQA heads).

    python tools/run_config4.py [modules=8] [sessions=1,2] [reps=2]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
SESS = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2").split(",")]
REPS = int(sys.argv[3]) if len(sys.argv) > 3 else 2
P, NEW = 32768, 256
cfg = LlamaConfig.llama8b(max_pos=P + NEW + 64)
base = ModuleWeights(cfg, 1, with_head=False)
mods = [ModuleWeights(cfg, 2 + i) for i in range(M)]
rng = np.random.default_rng(4)
for S in SESS:
    eng = PrefillShareEngine(cfg, M, S, P, NEW, pool_pages=S * (P // 16 + 1) + 64, modules=mods, base=base,
                             prefill_group=1)
    eng.capture()
    eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)])  # warm-up
    times, phases = [], []
    for _ in range(REPS):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)])
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
        phases.append(eng.last_phase_ms)
    t = min(times)
    print(json.dumps({"config": f"configs[3] on one GPU: 8B shape, {P}-token shared context, {M} decode modules, "
                                f"{NEW} tokens", "sessions": S, "requests_per_serve": S * M,
                      "req_per_s": round(S * M / t, 4), "serve_s": round(t, 3), "serves": [round(x, 3) for x in times],
                      "prefill_phase_ms": round(min(p["prefill"] for p in phases), 1),
                      "decode_phase_ms": round(min(p["decode"] for p in phases), 1),
                      "ms_per_token_step": round(min(p["decode"] for p in phases) / NEW, 3),
                      "weights_per_step_gb": round(M * mods[0].layer_bytes() / 1e9, 2) if hasattr(mods[0], "layer_bytes") else None,
                      "launches_per_step": eng.runner.launches_per_step}), flush=True)
    del eng
    torch.cuda.empty_cache()
