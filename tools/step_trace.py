"""K5-TC GEMV launch timeline inside the captured decode step (8B shape, 4
modules x S sessions): PSK_TRACE_RING=1 makes every CTA of every GEMV launch
stamp %globaltimer at entry, setup done, first TMA, PDL wait passed, last
TMA, last MMA commit, epilogue done and exit (psk_gemv_tc_trace_ring). Prints
one step's 129 GEMV launches of the last layers: per launch its N and grid,
phase medians / maxima after the launch's first CTA entry, its duration
(first entry -> last exit) and the gap from the previous GEMV's last exit.

    python tools/step_trace.py [S]
"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("PSK_TRACE_RING", "1")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2602_12029_b200 import _lib  # noqa: E402
from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
P, NEW = 4096, 256
cfg = LlamaConfig.llama8b(max_pos=P + NEW + 16)
eng = PrefillShareEngine(cfg, n_modules=4, max_sessions=S, max_prompt=P, max_new=NEW,
                         pool_pages=S * (P // 16 + 1) + 64, seed=0)
rng = np.random.default_rng(0)
eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)])
r = eng.runner
lib = _lib.load()
r.b.t_priv_len.fill_(NEW // 2)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
n0 = ctypes.c_int32()
stride = ctypes.c_int32()
with torch.cuda.stream(st):
    r._step(st.cuda_stream)
    st.synchronize()
    _lib.check(lib.psk_gemv_tc_trace_ring(None, 0, None, ctypes.byref(n0), ctypes.byref(stride)))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(2):
            r._step(st.cuda_stream)
    for _ in range(3):
        g.replay()
    st.synchronize()
n1 = ctypes.c_int32()
_lib.check(lib.psk_gemv_tc_trace_ring(None, 0, None, ctypes.byref(n1), ctypes.byref(stride)))
SL = 1024
buf = np.zeros(SL * stride.value * 8, dtype=np.uint64)
meta = np.zeros(2 * SL, dtype=np.int32)
_lib.check(lib.psk_gemv_tc_trace_ring(buf.ctypes.data, buf.size, meta.ctypes.data, ctypes.byref(n1),
                                      ctypes.byref(stride)))
ring = buf.reshape(SL, stride.value, 8).astype(np.int64)
per_step = (n1.value - n0.value) // 2
slots = [(n0.value + per_step + i) % SL for i in range(per_step)]  # the graph's second step
names = {cfg.qkv_dim: "qkv", 2 * cfg.ffn: "gate/up", cfg.vocab: "head"}
print(f"S={S}: {per_step} GEMV launches per step; columns: us after the launch's first CTA entry, median/max")
print("  #  kind     grid   setup        tma0        waited       tmaN        mma_done     epi_done     exit"
      "        dur    gap")
prev_exit = None
tot_gap = tot_dur = 0.0
for i, sl in enumerate(slots):
    N, grid = meta[2 * sl], meta[2 * sl + 1]
    live = ring[sl, :grid]
    t0 = live[:, 0].min()
    kind = names.get(N, "o/down" if N == cfg.d_model else str(N))
    cols = []
    for k in range(1, 8):
        v = live[:, k]
        v = v[v != 0]
        cols.append(f"{np.median(v - t0) / 1e3:5.1f}/{(v.max() - t0) / 1e3:5.1f}" if len(v) else "     -     ")
    ex = live[:, 7].max()
    dur = (ex - t0) / 1e3
    gap = None if prev_exit is None else (t0 - prev_exit) / 1e3
    prev_exit = ex
    tot_dur += dur
    if gap is not None:
        tot_gap += gap
    if i < 12 or i >= per_step - 5:
        print(f"{i:3d}  {kind:7s} {grid:4d}  " + "  ".join(cols) + f"  {dur:6.1f} " + ("" if gap is None else f"{gap:6.1f}"))
print(f"sum of GEMV launch durations {tot_dur:.0f} us, sum of gaps between consecutive GEMVs {tot_gap:.0f} us")
