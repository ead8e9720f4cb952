#!/bin/bash
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_attn_full_size_gpu.py -x -q -k "not k6" 2>&1 | tail -2
timeout 1200 python tools/k3_ab.py 4 4096 "new:" "old:PSK_LIB=paper_2602_12029_b200/var_oldk3.so" 2>&1 | tail -2
