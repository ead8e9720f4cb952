#!/bin/bash
for i in 1 2 3; do timeout 600 python -m pytest tests/test_staging_gpu.py -x -q 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
