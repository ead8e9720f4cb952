#!/bin/bash
# Round-2 late pass: full GPU suite, the default bench line, the launch list of
# one prefill + one decode step at the bench batch (default paths).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_step_launches_s32.csv python tools/profile_step.py 32 > /dev/null 2>&1; echo launches $?
