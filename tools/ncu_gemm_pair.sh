mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_pair -c 4 -o gpurun_out/ncu_gemm_pair -f python tools/profile_kernels.py gemm > gpurun_out/ncu_pair.log 2>&1
PSK_GEMM_PAIR=0 timeout 600 ncu --set full --clock-control none -k regex:gemm_bf16 -c 4 -o gpurun_out/ncu_gemm_1sm -f python tools/profile_kernels.py gemm > gpurun_out/ncu_1sm.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/ncu_pair.log
