#!/bin/bash
mkdir -p gpurun_out
free -g; nproc
timeout 900 python -m pytest tests/test_staging_gpu.py tests/test_serve.py -m gpu -x -q > gpurun_out/copy_tests.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/copy_tests.log
