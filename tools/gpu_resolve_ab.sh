nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for so in build/variants/*.so; do for r in 128 4096 65536; do for seed in 1234 1; do
 ROWS=$r SEED=$seed NODQ=1 F46_LIB_PATH=$so timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | tail -1 | sed "s|^|$so $r $seed |"; done; done; done
