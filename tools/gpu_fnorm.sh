#!/bin/bash
timeout 1200 python -m pytest tests/test_decode_gpu.py tests/test_fused_qkv_gpu.py tests/test_engine_gpu.py tests/test_full_parity_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for f in 1 0; do PSK_FUSED_NORM=$f timeout 600 python tools/step_ablation.py 32 quick 2>&1 | grep "full step"; done
done
