#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_attn_gpu.py tests/test_prefill_gpu.py tests/test_decode_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_attn.py 2>&1 | tail -5
timeout 400 python tools/bench_prefill.py 2>&1 | head -2
