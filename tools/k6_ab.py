"""K6 A/B at the fan-out shapes: the config-4 shape (32k shared tokens x 16
modules) and smaller fan-outs: the default (in-kernel merge, shared pages
streamed before the PDL wait) vs the PDL wait first (PSK_ATTN_LATE=1) vs the
merge kernel (PSK_ATTN_MERGE_KERNEL=1) vs the TMA stream alone, and against
another build of the library (PSK_LIB); env read once per process: one child
per mode.

    python tools/k6_ab.py [mode,mode,...]
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SHAPES = [(32767, 16, 1, 1), (32767, 8, 1, 1), (4095, 16, 1, 1), (4095, 16, 8, 16), (16383, 16, 2, 1)]
if os.environ.get("K6_SHAPES"):  # "shared:modules:sessions:priv,..."
    SHAPES = [tuple(int(v) for v in x.split(":")) for x in os.environ["K6_SHAPES"].split(",")]

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import bench
    peaks = bench._peaks()
    for shared, mods, sess, priv in SHAPES:
        r = bench.decode_attn_fanout(peaks, shared_tokens=shared, modules=mods, sessions=sess, priv=priv)
        print(json.dumps({"shared": shared, "modules": mods, "sessions": sess, "priv": priv,
                          "us": r["us_per_launch"], "gbs": r["achieved"], "frac": r["frac"]}), flush=True)
    sys.exit(0)

MODES = (("fused", {}),  # default: in-kernel merge, shared pages streamed before the PDL wait
         ("late", {"PSK_ATTN_LATE": "1"}),  # PDL wait before the first page
         ("merge-kernel", {"PSK_ATTN_MERGE_KERNEL": "1"}),
         ("stream-only", {"PSK_ATTN_STREAM_ONLY": "1"}),  # TMA stream alone, no MMA / softmax
         # A/B against another build of the library (variants/, tools/README.md)
         ("head", {"PSK_LIB": str(ROOT / "variants" / "libpsk_head.so")}),
         ("head-early", {"PSK_LIB": str(ROOT / "variants" / "libpsk_head.so"), "PSK_ATTN_EARLY": "1"}))
if len(sys.argv) > 1 and sys.argv[1] != "child":
    MODES = tuple(m for m in MODES if m[0] in sys.argv[1].split(","))
for mode, env in MODES:
    for rep in range(2):
        r = subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, **env), capture_output=True,
                           text=True, timeout=600)
        for line in r.stdout.splitlines():
            d = json.loads(line)
            print(f"{mode:13s} rep{rep} sessions={d['sessions']} shared={d['shared']:6d} modules={d['modules']:2d} "
                  f"priv={d['priv']:3d}: {d['us']:7.2f} us {d['gbs']:7.1f} GB/s ({d['frac']:.3f})", flush=True)
        if r.returncode:
            print(r.stderr[-2000:])
