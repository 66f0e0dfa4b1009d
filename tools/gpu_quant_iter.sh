# Quick quantize iteration on the GPU box: parity tests, K2 timings (variants), one ncu capture.
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
bash tools/gpu_variants.sh
python tools/time_quant.py fixed6 bf16
python tools/time_quant.py adaptive f32
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_seg -c 1 -o gpurun_out/quant_iter python tools/prof_quant.py > gpurun_out/ncu_iter.log 2>&1
