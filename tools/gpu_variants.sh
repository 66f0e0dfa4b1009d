# Time K1+K2 for every build/variants/*.so (adaptive bf16 on two seeds)
for so in build/variants/*.so; do
  F46_LIB_PATH=$so python tools/time_quant.py adaptive bf16
  SEED=1 F46_LIB_PATH=$so python tools/time_quant.py adaptive bf16
done
