#!/bin/bash
# All-heads kernel in-kernel merge: tests, A/B vs the previous build (bench shape), step time.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_attn_gpu.py -x -q -k "back_to_back or all_heads or fused_merge" > gpurun_out/k6_b2b.log 2>&1
echo "b2b/all-heads tests rc=$?"; tail -3 gpurun_out/k6_b2b.log
timeout 1200 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py tests/test_decode_gpu.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "attn/decode tests rc=$?"; tail -2 gpurun_out/k6_tests.log
export K6_SHAPES="4095:4:32:256,4095:4:32:1,4095:4:64:100,4095:1:148:1"
timeout 900 python tools/k6_ab.py fused,merge-kernel,head 2>&1
for i in 1 2 3; do
  echo "new: $(timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "old: $(PSK_LIB=variants/libpsk_head.so timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
done
