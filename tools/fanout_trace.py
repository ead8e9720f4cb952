"""K6 fan-out launch timeline across back-to-back launches (the bench's own
graph of 64 launches at the config-4 shape): every CTA stamps %globaltimer at
entry, barriers ready, first TMA issued, last TMA issued, partial written,
group merged and exit (PSK_TRACE_RING=1, psk_decode_attn_trace_ring). Prints
per-launch phase times (us after the launch's first CTA entry; median / max
over CTAs) and the gap from one launch's last exit to the next's first entry.

    PSK_TRACE_RING=1 python tools/fanout_trace.py [shared modules sessions priv]
"""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("PSK_TRACE_RING", "1")
import bench  # noqa: E402
from paper_2602_12029_b200 import _lib  # noqa: E402

args = [int(a) for a in sys.argv[1:5]] or [32767, 16, 1, 1]
peaks = bench._peaks()
r = bench.decode_attn_fanout(peaks, shared_tokens=args[0], modules=args[1], sessions=args[2], priv=args[3])
print(f"bench: {r['us_per_launch']} us/launch, frac {r['frac']}")
lib = _lib.load()
n, stride = ctypes.c_int32(), ctypes.c_int32()
_lib.check(lib.psk_decode_attn_trace_ring(None, 0, ctypes.byref(n), ctypes.byref(stride)))
slots = min(n.value, 512)
buf = np.zeros(slots * stride.value * 8, dtype=np.uint64)
_lib.check(lib.psk_decode_attn_trace_ring(buf.ctypes.data, buf.size, ctypes.byref(n), ctypes.byref(stride)))
ring = buf.reshape(slots, stride.value, 8).astype(np.int64)
names = ["entry", "bars", "tma0", "tmaN", "partial", "merged", "exit"]
# the last graph replay is the final len-64 run of slots (warm-up launches first)
last = [i for i in range(slots) if ring[i, 0, 0] != 0][-24:]
prev_exit = None
print("launch  " + "  ".join(f"{k:>13s}" for k in names) + "   gap(us)")
for i in last:
    live = ring[i][ring[i, :, 0] != 0]
    t0 = live[:, 0].min()
    cols = []
    for k in range(7):
        v = live[:, k]
        v = v[v != 0]
        cols.append(f"{np.median(v - t0) / 1e3:6.2f}/{(v.max() - t0) / 1e3:6.2f}" if len(v) else " " * 13)
    gap = "" if prev_exit is None else f"{(t0 - prev_exit) / 1e3:7.2f}"
    prev_exit = live[:, 6][live[:, 6] != 0].max() if (live[:, 6] != 0).any() else None
    print(f"{i:6d}  " + "  ".join(cols) + "   " + gap)
