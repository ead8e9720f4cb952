"""Sweep of the all-heads K6 split count (PSK_ATTN_HSPLIT is read once per
process, so each point runs in a child): sessions x splits -> us / layer."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if len(sys.argv) > 1 and sys.argv[1] == "one":
    sys.path.insert(0, str(ROOT))
    import bench  # noqa: E402
    sess = int(sys.argv[2])
    r = bench.decode_attn_fanout(bench._peaks(), shared_tokens=4095, modules=4, sessions=sess, priv=256, splits=None)
    print(f"sessions={sess:2d} hsplit={os.environ.get('PSK_ATTN_HSPLIT', 'auto'):>4s}: {r['us_per_launch']:8.2f} us "
          f"{r['achieved']:8.1f} GB/s ({r['frac']:.3f})", flush=True)
    sys.exit(0)
grid = {32: [0, 4, 5, 6, 7, 8], 64: [0, 2, 3, 4, 5, 6], 16: [0, 9, 12, 18], 8: [0, 18, 24, 36]}
for sess, hs in grid.items():
    for h in hs:
        env = dict(os.environ, PSK_ATTN_HSPLIT=str(h))
        subprocess.run([sys.executable, __file__, "one", str(sess)], env=env, check=True, timeout=300)
