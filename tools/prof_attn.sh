#!/bin/bash
# K6 profiling pass: per-CTA phase trace (PSK_TRACE), ncu full captures of the
# partial + merge kernels at the bench shape (8 sessions x 4k) and the fan-out
# shape (32k x 16 modules), and graph-timed latencies.
mkdir -p gpurun_out
for w in attn4k_s8 attn32k; do
  PSK_TRACE=1 timeout 300 python tools/profile_kernels.py $w > gpurun_out/trace_$w.txt 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 4 -c 2 \
    -o gpurun_out/ncu_$w -f python tools/profile_kernels.py $w > gpurun_out/ncu_$w.log 2>&1
  tail -1 gpurun_out/ncu_$w.log
done
tail -8 gpurun_out/trace_attn4k_s8.txt gpurun_out/trace_attn32k.txt
timeout 300 python tools/bench_attn.py 2>&1 | tail -6
