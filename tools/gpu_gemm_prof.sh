timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_nvfp4 -s 3 -c 1 -o gpurun_out/gemm_pair python tools/time_gemm.py 8192 8192 8192 bf16 > gpurun_out/ncu_gemm.log 2>&1
tail -2 gpurun_out/ncu_gemm.log
