#!/bin/bash
# One-GPU profiling pass for profiles/: bench JSON, per-kernel launch summary
# of a bench run, and full ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --print-summary per-kernel --csv \
  --log-file gpurun_out/launch_summary.csv python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 6 -c 1 -o gpurun_out/ncu_gemv python tools/profile_kernels.py gemv > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -c 2 -o gpurun_out/ncu_attn4k python tools/profile_kernels.py attn4k > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -c 2 -o gpurun_out/ncu_attn32k python tools/profile_kernels.py attn32k > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16|prefill_attn" -s 7 -c 6 -o gpurun_out/ncu_prefill python tools/profile_kernels.py gemm > /dev/null 2>&1
ls -la gpurun_out
