# GEMM timing probes (wrong results by design except g0): where the time goes
for so in build/variants/g*.so; do echo "== $so"; F46_LIB_PATH=$so timeout 120 python tools/time_gemm.py 8192 8192 8192 bf16 2>&1 | tail -1; F46_LIB_PATH=$so timeout 120 python tools/time_moe.py 2>&1 | tail -1; done
