#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_qkv_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for f in 1 0; do PSK_FUSED_QKV=$f timeout 600 python tools/step_ablation.py 32 quick 2>&1 | grep "full step"; done
done
timeout 600 ncu --set full --clock-control none -k regex:gemv_tc_kernel -s 1 -c 1 -o gpurun_out/ncu_r02_qkv_rope -f python tools/profile_kernels.py qkv_rope 32 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_r02_qkv_rope.ncu-rep
