#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "k6 tests rc=$?"; tail -3 gpurun_out/k6_tests.log
timeout 600 python tools/k6_ab.py 2>&1 | tee gpurun_out/k6_ab.log
export PSK_PARITY_OUT=gpurun_out/parity_full.json
timeout 1500 python -m pytest tests/test_full_parity_gpu.py -x -q -s > gpurun_out/parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/parity.log
