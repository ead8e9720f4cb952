#!/bin/bash
# correctness + quick perf pass for the current kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decode_attn_gpu.py tests/test_gemv_gpu.py tests/test_prefill_gpu.py tests/test_decode_gpu.py tests/test_gemm_gpu.py tests/test_transfer.py tests/test_serve.py -x -q 2>&1 | tail -15
for m in 1 4 8; do python tools/bench_gemv.py $m 2>&1 | cut -c1-90; done
PSK_TRACE=1 timeout 120 python tools/profile_kernels.py attn32k 2>&1 | tail -8
PSK_TRACE=1 timeout 120 python tools/profile_kernels.py attn4k 2>&1 | tail -8
