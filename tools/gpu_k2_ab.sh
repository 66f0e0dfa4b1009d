# K2 A/B: parity of the default build, then K2 timings of every variant on seeds with different tie directions
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_quant.py tests/test_gpu_fastpath_sweep.py tests/test_gpu_headline.py -x -q 2>&1 | tail -4
for so in build/variants/*.so; do
  for seed in ${SEEDS:-1234 1 2}; do SEED=$seed NODQ=1 F46_LIB_PATH=$so timeout 120 python tools/time_quant.py adaptive bf16 2>&1 | tail -1; done
done
