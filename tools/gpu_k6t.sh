#!/bin/bash
# K5-TC: weight boxes prefetched to L2 before the PDL wait (PSK_GEMV_L2PF = k-chunks) vs none.
PSK_GEMV_L2PF=24 timeout 900 python -m pytest tests/test_gemv_gpu.py -x -q 2>&1 | tail -1
for i in 1 2 3; do
  echo "pf0:  $(timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "pf12: $(PSK_GEMV_L2PF=12 timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "pf24: $(PSK_GEMV_L2PF=24 timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "pf48: $(PSK_GEMV_L2PF=48 timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
done
