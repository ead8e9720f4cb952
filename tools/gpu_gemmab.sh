#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_prefill_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
  echo "new: $(PSK_SEED=0 timeout 600 python tools/bench_prefill.py 4096 quick 2>&1 | grep 'prefill T')"
  echo "old: $(PSK_SEED=0 PSK_LIB=paper_2602_12029_b200/var_oldgemm.so timeout 600 python tools/bench_prefill.py 4096 quick 2>&1 | grep 'prefill T')"
done
timeout 900 python tools/prefill_group_ab.py 2 16 2>&1 | tail -1
PSK_LIB=paper_2602_12029_b200/var_oldgemm.so timeout 900 python tools/prefill_group_ab.py 2 16 2>&1 | tail -1
