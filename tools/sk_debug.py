"""Reproduce one K6 stream-K test case outside pytest (for compute-sanitizer)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import test_decode_attn_gpu as t  # noqa: E402

case = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cases = [(32, 8, [4095], [4], [0, 3, 17, 255]), (32, 8, [4095] * 8, [4] * 8, [255] * 32),
         (32, 8, [1000, 37, 513], [2, 3, 1], [0, 5, 16, 40, 1, 200])]
nq, nkv, lens, rps, priv = cases[case]
t._case(nq, nkv, lens, rps, priv, 0, seed=len(lens))
print("ok", case)
