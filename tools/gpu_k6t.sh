#!/bin/bash
# All-heads kernel: first stages streamed before the PDL wait. Tests + in-step A/B (PSK_ATTN_LATE=1 = off).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_decode_attn_gpu.py tests/test_decode_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "attn/decode tests rc=$?"; tail -2 gpurun_out/k6_tests.log
for i in 1 2 3 4; do
  echo "early: $(timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "late:  $(PSK_ATTN_LATE=1 timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
done
