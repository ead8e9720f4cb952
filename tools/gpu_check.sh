#!/bin/bash
# correctness + perf pass: GPU tests, per-launch list of one bench step,
# full ncu captures of the three hot kernels, bench line.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
S=${S:-8}
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/step_launches_s$S.csv python tools/profile_step.py $S > gpurun_out/profile_step.log 2>&1
tail -1 gpurun_out/profile_step.log
for m in 1 8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 \
    -o gpurun_out/ncu_gemv_m$m -f python tools/profile_kernels.py gemv $m > gpurun_out/ncu_gemv_m$m.log 2>&1
  tail -1 gpurun_out/ncu_gemv_m$m.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn_partial -s 2 -c 1 \
  -o gpurun_out/ncu_attn4k_s8 -f python tools/profile_kernels.py attn4k_s8 > gpurun_out/ncu_attn4k_s8.log 2>&1
tail -1 gpurun_out/ncu_attn4k_s8.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn_pp -s 2 -c 1 \
  -o gpurun_out/ncu_prefill_attn -f python tools/profile_kernels.py prefill_attn > gpurun_out/ncu_prefill_attn.log 2>&1
tail -1 gpurun_out/ncu_prefill_attn.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 5000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
