#!/bin/bash
# A/B the default lib against variants/*.so on the K6 fan-out shapes, alternating.
for rep in 1 2; do
  echo "== default"; timeout 300 python tools/bench_attn.py 2>&1 | tail -6
  for v in variants/*.so; do echo "== $v"; PSK_LIB=$v timeout 300 python tools/bench_attn.py 2>&1 | tail -6; done
done
