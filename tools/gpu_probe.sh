#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_attn_gpu.py tests/test_decode_gpu.py -x -q 2>&1 | tail -2
PSK_TRACE=1 timeout 120 python tools/profile_kernels.py attn4k_s8 2>&1 | grep -E "staged|loop-done|folded" | tail -3
timeout 300 python tools/bench_attn.py 2>&1 | tail -5
