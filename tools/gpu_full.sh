#!/bin/bash
# Full pass: GPU tests (incl. full-size parity), bench (ours), reference arm.
mkdir -p gpurun_out
export PSK_PARITY_OUT=gpurun_out/parity_full.json
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -c 800 gpurun_out/bench_ref.json
