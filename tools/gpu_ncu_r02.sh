#!/bin/bash
# Round-2 ncu captures (--set full, cold cache, serialised): K6 (bench shape,
# config-4 fan-out), the fused decode QKV (+RoPE/append) GEMV, the prefill QKV
# GEMM with its RoPE + paged-KV epilogue, K3, the K8 page copy; plus the
# launch list of one prefill + one decode step at 32 sessions.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:decode_attn -c 2 -o gpurun_out/ncu_r02_attn32k -f python tools/profile_kernels.py attn32k > /dev/null 2>&1; echo attn32k $?
timeout 600 $N -k regex:decode_attn -c 4 -o gpurun_out/ncu_r02_attn4k_s32 -f python tools/profile_kernels.py attn4k_s32 > /dev/null 2>&1; echo attn4k $?
timeout 600 $N -k regex:gemv_tc_kernel -s 1 -c 1 -o gpurun_out/ncu_r02_qkv_rope -f python tools/profile_kernels.py qkv_rope 32 > /dev/null 2>&1; echo qkv_rope $?
timeout 600 $N -k regex:"gemm_pair|prefill_attn_pp" -c 5 -o gpurun_out/ncu_r02_prefill -f python tools/profile_kernels.py gemm > /dev/null 2>&1; echo prefill $?
timeout 600 $N -k regex:copy_pages -s 1 -c 1 -o gpurun_out/ncu_r02_kvcopy -f python tools/profile_kernels.py kvcopy > /dev/null 2>&1; echo kvcopy $?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_step_launches_s32.csv python tools/profile_step.py 32 > /dev/null 2>&1; echo launches $?
for f in gpurun_out/ncu_r02_*.ncu-rep; do python tools/ncu_summary.py $f; done > gpurun_out/ncu_r02_summary.txt 2>&1
cat gpurun_out/ncu_r02_summary.txt
