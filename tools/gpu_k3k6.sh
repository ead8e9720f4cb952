#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_k3.sh 2>&1 | tee gpurun_out/k3.log
timeout 900 python -m pytest tests/test_decode_attn_gpu.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "k6 tests rc=$?"; tail -3 gpurun_out/k6_tests.log
timeout 600 python tools/k6_ab.py 2>&1 | tee gpurun_out/k6_ab.log
PSK_TRACE=1 timeout 300 python tools/profile_kernels.py attn32k 2>&1 | tail -8
