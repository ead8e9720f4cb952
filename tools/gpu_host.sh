#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_disagg_gpu.py tests/test_serve.py tests/test_staging_gpu.py tests/test_pool.py tests/test_engine_gpu.py -m gpu -x -q > gpurun_out/host_tests.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/host_tests.log
timeout 900 python tools/run_agents.py --shape tiny --sweep arrival_rate --values 2,4 --auto-concurrency --cap-grid 10,20 --duration 3 --rows 8 --pool-pages 1024 --out gpurun_out/sweep_tiny > gpurun_out/sweep_tiny.log 2>&1
echo "sweep rc=$?"; tail -8 gpurun_out/sweep_tiny.log
