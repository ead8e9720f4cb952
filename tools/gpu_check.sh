#!/bin/bash
# correctness + perf pass: GPU tests, GEMV sweep, per-launch list of one
# bench step, one full ncu capture of the gate/up GEMV, and the bench line.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for m in 1 4 8 16; do timeout 300 python tools/bench_gemv.py $m 2>&1 | cut -c1-90; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/step_launches.csv python tools/profile_step.py 1 > gpurun_out/profile_step.log 2>&1
tail -2 gpurun_out/profile_step.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_gemv -f python tools/profile_kernels.py gemv > gpurun_out/ncu_gemv.log 2>&1
tail -2 gpurun_out/ncu_gemv.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
