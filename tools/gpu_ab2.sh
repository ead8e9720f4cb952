#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/k3_ab.py 6 2>&1 | tee gpurun_out/k3_ab.log
timeout 600 python tools/k6_ab.py 2>&1 | tee gpurun_out/k6_ab.log
PSK_ATTN_EARLY=1 PSK_TRACE=1 timeout 300 python tools/profile_kernels.py attn32k 2>&1 | tail -7
