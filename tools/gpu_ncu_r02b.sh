#!/bin/bash
# Round-2 late ncu captures (--set full, cold cache, serialised) of the changed
# K6 kernels: the all-heads kernel with its in-kernel merge (bench shape) and
# the fan-out kernel (config 4).
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:decode_attn -c 2 -o gpurun_out/ncu_r02b_attn32k -f python tools/profile_kernels.py attn32k > /dev/null 2>&1; echo attn32k $?
timeout 600 $N -k regex:decode_attn -c 2 -o gpurun_out/ncu_r02b_attn4k_s32 -f python tools/profile_kernels.py attn4k_s32 > /dev/null 2>&1; echo attn4k $?
for f in gpurun_out/ncu_r02b_*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/ncu_r02b_summary.txt 2>&1
cat gpurun_out/ncu_r02b_summary.txt
