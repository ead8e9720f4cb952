"""Serve-level A/B of the prefill group size (sessions whose prefills share
one batched forward): 32 fresh 4096-token prompts per serve, 4 modules,
max_new tokens, device time of the prefill phase (engine.last_phase_ms).

    python tools/prefill_group_ab.py [groups, e.g. 1,2,4] [max_new]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights  # noqa: E402

groups = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,4").split(",")]
NEW = int(sys.argv[2]) if len(sys.argv) > 2 else 16
S, P = 32, 4096
cfg = LlamaConfig.llama8b(max_pos=P + NEW + 64)
base = ModuleWeights(cfg, 1, with_head=False)
mods = [ModuleWeights(cfg, 2 + i) for i in range(4)]
rng = np.random.default_rng(0)
res = {}
for rep in range(2):
    for gsz in groups:
        eng = PrefillShareEngine(cfg, 4, S, P, NEW, pool_pages=3 * S * (P // 16 + 1), modules=mods, base=base,
                                 prefill_group=gsz)
        eng.capture() if hasattr(eng, "capture") else None
        for _ in range(2):
            eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)])
        t = []
        for _ in range(3):
            eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)])
            t.append(eng.last_phase_ms["prefill"])
        res.setdefault(gsz, []).extend(t)
        print(f"rep {rep} group {gsz}: prefill phase {min(t):.1f} ms (min of 3), runs {[round(x, 1) for x in t]}",
              flush=True)
        del eng
        torch.cuda.empty_cache()
for gsz, v in res.items():
    print(f"group {gsz}: best {min(v):.1f} ms, median {sorted(v)[len(v) // 2]:.1f} ms per 32-prompt serve")
