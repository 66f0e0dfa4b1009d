# config-2 weights (fused amax+quantize), C1 fixed6/adaptive, K2 at three sizes, for each variant
for so in build/variants/*.so; do echo "== $so"; F46_LIB_PATH=$so python tools/time_weights.py 2>&1 | tail -1
  F46_LIB_PATH=$so python tools/time_c1.py 2>&1 | tail -1
  for r in 128 4096 65536; do ROWS=$r NODQ=1 F46_LIB_PATH=$so timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | tail -1; done; done
