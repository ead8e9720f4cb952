#!/bin/bash
# Round pass: GPU tests, bench line, launch list of one prefill + one decode
# step at the bench batch, ncu full captures of the hot kernels.
mkdir -p gpurun_out
S=${S:-32}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/step_launches_s$S.csv python tools/profile_step.py $S > gpurun_out/profile_step.log 2>&1
tail -1 gpurun_out/profile_step.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_gemv_tc_m$((S)) -f python tools/profile_kernels.py gemv_tc $S > gpurun_out/ncu_gemv_tc.log 2>&1
tail -1 gpurun_out/ncu_gemv_tc.log
