"""Feasibility probe: prefill of the next batch beside decode of the current
one, each on its own stream with a share of the SMs (psk_set_sm_budget).

    python tools/overlap_probe.py D:P [D:P ...]   (decode / prefill SM budgets)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2602_12029_b200 import _lib  # noqa: E402
from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig  # noqa: E402

pairs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]] or [(148, 148)]
D, P = pairs[0]
NP, ND = 4, 64   # prefills, decode steps per measurement
cfg = LlamaConfig.llama8b(max_pos=4096 + 256 + 64)
_lib.set_sm_budget(D)
eng = PrefillShareEngine(cfg, 4, 32, 4096, 256, pool_pages=2 * 32 * 257 + 64, seed=1)
eng.capture()
toks = torch.randint(0, cfg.vocab, (4096,), device="cuda")
pt = torch.arange(257, dtype=torch.int32, device="cuda")
import os  # noqa: E402
if os.environ.get("PROBE_NO_ATTN"):  # K3 grids are not budgeted: no-op them to isolate the GEMMs
    eng.prefill.lib.psk_prefill_attn = lambda *a: 0
sD = torch.cuda.Stream(priority=-1)
sP = torch.cuda.Stream(priority=0)
g = eng.runner.graph


def decode():
    g = eng.runner.graph
    with torch.cuda.stream(sD):
        for _ in range(ND):
            g.replay()


def prefill():
    _lib.set_sm_budget(P)
    with torch.cuda.stream(sP):
        for _ in range(NP):
            eng.prefill.run(toks, 0, pt, stream=sP.cuda_stream)
    _lib.set_sm_budget(D)


def timed(fn_list, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sD.wait_event(e0)
        sP.wait_event(e0)
        for f in fn_list:
            f()
        torch.cuda.current_stream().wait_stream(sD)
        torch.cuda.current_stream().wait_stream(sP)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for D, P in pairs:
    _lib.set_sm_budget(D)
    eng.capture()
    g = eng.runner.graph
    decode(); prefill(); torch.cuda.synchronize()
    td = timed([decode])
    tp = timed([prefill])
    tb = timed([prefill, decode])
    print(f"D={D} P={P}: decode {ND} steps {td:.1f} ms ({td / ND * 1e3:.0f} us/step) | prefill x{NP} {tp:.1f} ms "
          f"({tp / NP:.1f} ms each) | both {tb:.1f} ms vs sum {td + tp:.1f} (overlap saves {td + tp - tb:.1f})",
          flush=True)
