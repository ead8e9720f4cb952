#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_disagg_gpu.py tests/test_serve.py tests/test_staging_gpu.py tests/test_pool.py tests/test_engine_gpu.py -m gpu -x -q > gpurun_out/host_tests.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/host_tests.log
