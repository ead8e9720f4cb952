#!/bin/bash
# Round 2, pass A: full-size parity tests (bench config through the engine,
# K3 at 4k, K6 at 32k x 16) + ncu captures of the current K6 kernels.
mkdir -p gpurun_out
export PSK_PARITY_OUT=gpurun_out/parity_full.json
timeout 1500 python -m pytest tests/test_attn_full_size_gpu.py tests/test_full_parity_gpu.py -x -q -s \
  > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; tail -5 gpurun_out/parity.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -c 4 \
  -o gpurun_out/ncu_attn4k_s32 -f python tools/profile_kernels.py attn4k_s32 > gpurun_out/ncu_attn4k.log 2>&1
tail -1 gpurun_out/ncu_attn4k.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -c 4 \
  -o gpurun_out/ncu_attn32k -f python tools/profile_kernels.py attn32k > gpurun_out/ncu_attn32k.log 2>&1
tail -1 gpurun_out/ncu_attn32k.log
