"""Time K6 (decode attention) at fan-out shapes, graph-replayed over 32
layers (working set > L2). Set PSK_ATTN_TC=1 to use the tcgen05 fan-out path.

    python tools/bench_attn.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402

peaks = {"hbm": 6539.2}
for shared, mods in [(4095, 4), (4095, 16), (32767, 4), (32767, 8), (32767, 16)]:
    r = bench.decode_attn_fanout(peaks, shared_tokens=shared, modules=mods)
    print(f"shared={shared:6d} modules={mods:3d}: {r['us_per_launch']:8.2f} us "
          f"{r['achieved']:8.1f} GB/s ({r['frac']:.3f})", flush=True)
