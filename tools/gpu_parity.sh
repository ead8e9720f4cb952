#!/bin/bash
mkdir -p gpurun_out
export PSK_PARITY_OUT=gpurun_out/parity_full.json
timeout 1500 python -m pytest tests/test_full_parity_gpu.py -x -q -s > gpurun_out/parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/parity.log
