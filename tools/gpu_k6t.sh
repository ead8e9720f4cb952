#!/bin/bash
# Stream-K all-heads kernel (PSK_ATTN_HEADS_SK=1): tests, A/B, step time.
mkdir -p gpurun_out
PSK_ATTN_HEADS_SK=1 timeout 900 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py tests/test_decode_gpu.py -x -q -k "all_heads or bench_shape or decode" > gpurun_out/hsk_tests.log 2>&1
echo "hsk tests rc=$?"; tail -3 gpurun_out/hsk_tests.log
export K6_SHAPES="4095:4:32:256,4095:4:32:1,4095:4:64:100,4095:1:148:1,700:1:200:30"
timeout 900 python tools/k6_ab.py fused,heads-sk 2>&1 | grep -v "^ \|Trace\|^$"
for i in 1 2 3; do
  echo "hk:  $(timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "hsk: $(PSK_ATTN_HEADS_SK=1 timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
done
