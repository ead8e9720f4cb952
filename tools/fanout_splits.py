"""K6 fan-out at the config-4 shape (32k shared tokens x 16 modules) over the
split count per KV head (one wave needs splits x 8 <= 148): bench.decode_attn_fanout.

    python tools/fanout_splits.py [splits,...]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

peaks = bench._peaks()
for ns in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "18,17,16,14,12").split(",")]:
    for rep in range(2):
        r = bench.decode_attn_fanout(peaks, splits=ns)
        print(json.dumps({"splits": ns, "rep": rep, "us": r["us_per_launch"], "frac": r["frac"]}), flush=True)
