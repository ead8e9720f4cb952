"""TinyLM evaluateSharing timing alone (bench.tinylm_point): GPU
psk_tiny_forward path vs the CPU oracle on the same call.

    python tools/tinylm_time.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

print(json.dumps(bench.tinylm_point()))
