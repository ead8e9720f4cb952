#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemv_gpu.py tests/test_decode_gpu.py -x -q 2>&1 | tail -2
for m in 1 8 16; do timeout 300 python tools/bench_gemv.py $m 2>&1 | cut -c1-90; done
timeout 400 python tools/step_ablation.py 8 2>&1 | head -1
