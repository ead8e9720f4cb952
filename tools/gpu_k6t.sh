#!/bin/bash
PSK_ATTN_HK_INTERLEAVE=1 timeout 600 python -m pytest tests/test_decode_attn_gpu.py -x -q -k "all_heads" 2>&1 | tail -1
export K6_SHAPES="4095:4:32:256,4095:4:32:1,4095:4:64:100"
timeout 900 python tools/k6_ab.py fused,interleave 2>&1
