"""Time K6 (decode attention) at fan-out shapes, graph-replayed over 32
layers (working set > L2). Set PSK_ATTN_TC=1 to use the tcgen05 fan-out path.

    python tools/bench_attn.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402

peaks = bench._peaks()
for shared, mods, sess, priv in [(4095, 4, 8, 256), (4095, 4, 32, 256), (4095, 4, 1, 1), (4095, 16, 1, 1),
                                 (32767, 4, 1, 1), (32767, 8, 1, 1), (32767, 16, 1, 1)]:
    for splits in (None, 0):
        r = bench.decode_attn_fanout(peaks, shared_tokens=shared, modules=mods, sessions=sess, priv=priv,
                                     splits=splits)
        print(f"{'stream-K' if splits == 0 else 'fixed   '} sessions={sess:2d} shared={shared:6d} modules={mods:3d} "
              f"priv={priv:4d}: {r['us_per_launch']:8.2f} us {r['achieved']:8.1f} GB/s ({r['frac']:.3f})",
              flush=True)
