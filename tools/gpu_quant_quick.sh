# Quantize iteration: GPU parity tests of K2 paths, K1/K2 timings on two seeds.
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | grep K2
SEED=1 timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | grep K2
timeout 120 python tools/time_quant.py fixed6 bf16 2>&1 | grep K2
timeout 120 python tools/time_quant.py adaptive f32 2>&1 | grep K2
