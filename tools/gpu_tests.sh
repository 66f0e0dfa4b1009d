set -x
timeout 900 python -m pytest tests/test_gpu_linear.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
