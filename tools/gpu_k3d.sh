#!/bin/bash
timeout 300 python -m pytest tests/test_prefill_gpu.py tests/test_attn_full_size_gpu.py -x -q -k "not k6 and not variant" 2>&1 | tail -1
PSK_LIB=paper_2602_12029_b200/var_dyn.so timeout 240 python -m pytest tests/test_prefill_gpu.py tests/test_attn_full_size_gpu.py -x -q -k "not k6 and not variant" 2>&1 | tail -1
rc=${PIPESTATUS[0]}
if [ "$rc" = "0" ]; then timeout 900 python tools/k3_ab.py 4 4096 "base:" "dyn:PSK_LIB=paper_2602_12029_b200/var_dyn.so" 2>&1 | tail -2; fi
