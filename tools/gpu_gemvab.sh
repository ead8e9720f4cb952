#!/bin/bash
for rep in 1 2 3; do
  echo "new: $(timeout 600 python tools/step_ablation.py 32 quick 2>&1 | grep 'full step')"
  echo "old: $(PSK_LIB=paper_2602_12029_b200/var_oldgemv.so timeout 600 python tools/step_ablation.py 32 quick 2>&1 | grep 'full step')"
done
