#!/bin/bash
PSK_ATTN_HEADS_SK=1 timeout 900 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py -x -q -k "all_heads or bench_shape or stream_k or multi_session or ragged" 2>&1 | tail -2
K6_SHAPES="4095:4:32:256,4095:4:20:1,4095:4:64:100,2047:4:40:1,4095:1:148:1" timeout 900 python tools/k6_ab.py fused,heads-sk 2>&1 | grep -v "^$"
