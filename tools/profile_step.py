"""One 8B-shape prefill (4k prompt) + one decode step (4 modules x S sessions),
eager, inside a cudaProfilerStart/Stop range — the per-launch list of the
bench step for ncu:

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/step_launches.csv \
        python tools/profile_step.py [S]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1
P, NEW = 4096, 256
cfg = LlamaConfig.llama8b(max_pos=P + NEW + 16)
eng = PrefillShareEngine(cfg, n_modules=4, max_sessions=S, max_prompt=P, max_new=NEW,
                         pool_pages=S * (P // 16) + 64, seed=0)
rng = np.random.default_rng(0)
prompts = [rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)]
eng.serve(prompts)  # warm: graph capture, kernel attributes, pool state
torch.cuda.synchronize()
toks = torch.from_numpy(prompts[0]).cuda()
pt = torch.arange(P // 16, dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
torch.cuda.profiler.start()
eng.prefill.run(toks, 0, pt)
eng.runner._step(stream)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled: 1 prefill call + 1 decode step, sessions", S)
