# WGRAD-operand kernels: parity + timing (default build vs build/variants/*.so)
timeout 600 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_sr_rht.py -x -q 2>&1 | tail -3
python tools/time_rht.py 2>&1 | tail -3
for so in build/variants/*.so; do echo "== $so"; F46_LIB_PATH=$so python tools/time_rht.py 2>&1 | tail -3; done
