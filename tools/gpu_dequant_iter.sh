# Dequantize iteration: parity tests touching K3, K3 timings (both variants), calibration.
set -x
timeout 600 python -m pytest tests/test_gpu_quant.py -x -q 2>&1 | tail -3
timeout 120 python tools/time_dequant.py
F46_DQ_VEC=1 timeout 120 python tools/time_dequant.py
