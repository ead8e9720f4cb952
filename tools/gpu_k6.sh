#!/bin/bash
# K6 fan-out: tests, A/B timing, ncu capture of the tcgen05 kernel at 32k x 16.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_attn_gpu.py tests/test_attn_full_size_gpu.py -x -q > gpurun_out/k6_tests.log 2>&1
echo "k6 tests rc=$?"; tail -3 gpurun_out/k6_tests.log
timeout 600 python tools/k6_ab.py 2>&1 | tee gpurun_out/k6_ab.log
PSK_TRACE=1 timeout 300 python tools/profile_kernels.py attn32k > gpurun_out/k6_trace.log 2>&1; tail -20 gpurun_out/k6_trace.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -c 2 \
  -o gpurun_out/ncu_attn32k_r02 -f python tools/profile_kernels.py attn32k > gpurun_out/ncu_attn32k.log 2>&1
tail -1 gpurun_out/ncu_attn32k.log
