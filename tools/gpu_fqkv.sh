#!/bin/bash
# Fused QKV (RoPE + KV append in the K5-TC epilogue): parity tests, then the
# decode step A/B (PSK_FUSED_QKV=1/0) and the default bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_qkv_gpu.py tests/test_decode_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/fqkv_tests.log 2>&1
echo "fqkv tests rc=$?"; tail -3 gpurun_out/fqkv_tests.log
for rep in 1 2; do
  for f in 1 0; do echo "== PSK_FUSED_QKV=$f"; PSK_FUSED_QKV=$f timeout 600 python tools/step_ablation.py 32 quick 2>&1 | grep "full step"; done
done
timeout 900 python tools/fanout_insitu.py 4 16 32768 2>&1 | tail -2
