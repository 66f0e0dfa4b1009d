set -x
timeout 300 python -m pytest tests/test_gpu_quant.py -x -q -k dequant 2>&1 | tail -2
for so in build/variants/*.so; do echo $so; F46_LIB_PATH=$so timeout 120 python tools/time_dequant.py 2>&1 | head -2; done
