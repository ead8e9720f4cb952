#!/bin/bash
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_fused_qkv_gpu.py -x -q 2>&1 | tail -1
timeout 900 python tools/step_trace.py 32 2>&1 | tail -22
