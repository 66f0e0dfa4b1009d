set -x
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -15
timeout 120 python tools/time_gemm.py
timeout 120 python tools/time_gemm.py 8192 8192 8192 bf16
F46_GEMM_1SM=1 timeout 120 python tools/time_gemm.py 8192 8192 8192 bf16
timeout 120 python tools/time_gemm.py 3072 2688 1856
