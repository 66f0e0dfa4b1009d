bash tools/gpu_variants.sh
