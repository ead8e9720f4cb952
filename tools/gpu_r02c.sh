#!/bin/bash
# Round 2 (re-entry): full GPU suite + default bench line on the current build.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
