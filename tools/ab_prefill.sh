#!/bin/bash
# A/B the default lib against variants/*.so on the 4k prefill and its K3 attention, alternating.
for rep in 1 2; do
  echo "== default"; timeout 300 python tools/bench_prefill.py 4096 attn 2>&1 | tail -2
  for v in variants/*.so; do echo "== $v"; PSK_LIB=$v timeout 300 python tools/bench_prefill.py 4096 attn 2>&1 | tail -2; done
done
