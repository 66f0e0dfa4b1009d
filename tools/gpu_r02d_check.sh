# full GPU suite + K2 timings at three sizes with the default build
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for r in 128 4096 65536; do for seed in 1234 1; do
 ROWS=$r SEED=$seed NODQ=1 timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | tail -1; done; done
