#!/bin/bash
# K6 fan-out: generation-counter merge barrier; tests (incl. back-to-back stress) and A/B.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_attn_gpu.py -x -q -k "back_to_back or fused_merge" > gpurun_out/k6_b2b.log 2>&1
echo "b2b tests rc=$?"; tail -3 gpurun_out/k6_b2b.log
timeout 900 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "k6 tests rc=$?"; tail -2 gpurun_out/k6_tests.log
export K6_SHAPES="32767:16:1:1,4095:16:8:16,16383:16:2:1,4095:16:4:200,4095:16:1:1"
timeout 900 python tools/k6_ab.py fused,head-early 2>&1
timeout 300 python tools/fanout_trace.py 2>&1 | tail -4
