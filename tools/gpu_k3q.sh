#!/bin/bash
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_attn_full_size_gpu.py tests/test_evaluate_gpu.py -x -q -k "not k6" 2>&1 | tail -2
PSK_PREFILL_SPLIT=1 timeout 900 python -m pytest tests/test_attn_full_size_gpu.py -x -q -k "k3" 2>&1 | tail -1
PSK_PREFILL_QT=1 timeout 900 python -m pytest tests/test_attn_full_size_gpu.py -x -q -k "k3" 2>&1 | tail -1
timeout 1500 python tools/k3_ab.py 3 4096 "qt:" "smemq:PSK_PREFILL_QT=0" "smemq-mma-only:PSK_PREFILL_QT=0;PSK_PREFILL_MMA_ONLY=1" "smemq-split1:PSK_PREFILL_SPLIT=1;PSK_PREFILL_QT=0" 2>&1 | tail -4
