#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_prefill.py 2>&1 | tail -2
PSK_PREFILL_TC1=1 timeout 300 python tools/bench_prefill.py 2>&1 | tail -2
