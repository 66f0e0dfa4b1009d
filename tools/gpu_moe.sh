F46_LIB_PATH=build/variants/diag.so timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
for so in build/variants/*.so; do echo $so; F46_LIB_PATH=$so timeout 120 python tools/time_moe.py | tail -1; F46_LIB_PATH=$so timeout 120 python tools/time_gemm.py 8192 8192 8192 bf16; done
