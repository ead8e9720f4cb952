#!/bin/bash
# K3: parity tests (prefill / full-size K3), then A/B of the TMEM-P kernel
# (default) vs the shared-memory-P kernel (PSK_PREFILL_PSMEM=1), alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_attn_full_size_gpu.py -x -q -k "not k6" > gpurun_out/k3_tests.log 2>&1
echo "k3 tests rc=$?"; tail -3 gpurun_out/k3_tests.log
for rep in 1 2 3; do
  echo "== tmem-P"; timeout 300 python tools/bench_prefill.py 4096 attn 2>&1 | tail -2
  echo "== smem-P"; PSK_PREFILL_PSMEM=1 timeout 300 python tools/bench_prefill.py 4096 attn 2>&1 | tail -2
done
