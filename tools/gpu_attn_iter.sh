#!/bin/bash
# K6 iteration: GPU tests, graph-timed latencies, per-CTA phase traces.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/bench_attn.py 2>&1 | tail -6
for w in attn4k_s8 attn32k; do
  PSK_TRACE=1 timeout 300 python tools/profile_kernels.py $w 2>&1 | tail -7
done
