"""Time the tcgen05 NVFP4 GEMM with CUDA events.  Usage: python tools/time_gemm.py [M N K] [bf16]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 8192, 8192)
od = torch.bfloat16 if "bf16" in sys.argv else torch.float32
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
cfg = f46.QuantConfig(scale_mode="adaptive")
aq = f46.quantize_tensor_adaptive(torch.randn(M, K, generator=g, device=dev).to(torch.bfloat16), cfg)
bq = f46.quantize_tensor_adaptive(torch.randn(N, K, generator=g, device=dev).to(torch.bfloat16), cfg)
out = torch.empty((M, N), dtype=od, device=dev)
for _ in range(3):
    f46.gemm_nvfp4(aq, bq, od, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f46.gemm_nvfp4(aq, bq, od, out=out); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = sorted(ts)[len(ts) // 2]
print(f"gemm {M}x{N}x{K} {od}: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TFLOP/s")
# back to back (as the vendor comparison tools/time_torch_fp4.py times it)
reps = 10
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
torch.cuda._sleep(1_000_000)
a.record()
for _ in range(reps):
    f46.gemm_nvfp4(aq, bq, od, out=out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"gemm {M}x{N}x{K} {od} back-to-back: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TFLOP/s")
