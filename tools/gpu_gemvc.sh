#!/bin/bash
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_decode_gpu.py tests/test_fused_qkv_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do timeout 600 python tools/step_ablation.py 32 quick 2>&1 | grep "full step"; done
timeout 600 python tools/bench_gemv.py 32 tc 2>&1 | tail -12
