#!/bin/bash
PSK_ATTN_TC_STAGES=3 timeout 600 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py -x -q -k "fanout or growing or sixteen" 2>&1 | tail -2
timeout 900 python tools/k6_ab.py fused,overlap3,overlap3-stream-only
PSK_ATTN_TC_STAGES=3 PSK_TRACE=1 timeout 300 python tools/profile_kernels.py attn32k 2>&1 | tail -7
