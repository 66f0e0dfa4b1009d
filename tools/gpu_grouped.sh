# grouped quantization: parity tests, C5 headline tests, MoE step timing
timeout 900 python -m pytest tests/test_gpu_grouped.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -k "c5" 2>&1 | tail -3
timeout 600 python - <<'PY'
import sys, torch, json
sys.path.insert(0, ".")
import bench
dev = torch.device("cuda", 0)
class A: pass
r = bench.bench_moe(A(), dev)
print(json.dumps({k: v for k, v in r.items() if k != "per_gemm"}, indent=1))
PY
