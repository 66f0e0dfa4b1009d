# K2 alone and the fused path across sizes, with and without the parallel-resolver instantiation
for so in build/variants/*.so; do echo "== $so"; for r in 4096 6144 8192 12288; do ROWS=$r NODQ=1 F46_LIB_PATH=$so timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | tail -1 | sed "s/^/$r /"; done
F46_LIB_PATH=$so python tools/time_fused_sizes.py 2>&1 | tail -4; done
