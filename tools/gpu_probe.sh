#!/bin/bash
# HBM read-pattern probe, GEMV sweep, GEMV/attention parity
mkdir -p gpurun_out
timeout 300 tools/_bin/bw_probe
timeout 600 python -m pytest tests/test_gemv_gpu.py tests/test_decode_gpu.py tests/test_decode_attn_gpu.py -x -q 2>&1 | tail -3
for m in 1 4 8 16; do timeout 300 python tools/bench_gemv.py $m 2>&1 | cut -c1-90; done
