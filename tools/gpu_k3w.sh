#!/bin/bash
timeout 900 python -m pytest tests/test_prefill_gpu.py tests/test_attn_full_size_gpu.py tests/test_evaluate_gpu.py -x -q -k "not k6" 2>&1 | tail -2
timeout 1500 python tools/k3_ab.py 3 4096 "kc128:" "kc64:PSK_PREFILL_KC64=1" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none -k regex:prefill_attn -s 2 -c 1 -o gpurun_out/ncu_r02_k3_kc128 -f python tools/profile_kernels.py prefill_attn > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_r02_k3_kc128.ncu-rep
