#!/bin/bash
mkdir -p gpurun_out

timeout 400 python tools/bench_prefill.py 2>&1 | tail -12

