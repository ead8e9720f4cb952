#!/bin/bash
# K5-TC at 32 rows/module: 2 k-chunks per stage x 5 stages (variants/libpsk_ch2.so) vs 3 x 3 (default).
for i in 1 2 3; do
  echo "ch3: $(timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
  echo "ch2: $(PSK_LIB=variants/libpsk_ch2.so timeout 600 python tools/step_ablation.py 32 quick 2>&1 | tail -1)"
done
