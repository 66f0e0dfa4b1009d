"""Vendor-library comparison for the GEMM roofline: torch._scaled_mm on NVFP4
operands (cuBLASLt block-scaled FP4, e2m1 + 16-element e4m3 scales) at
8192^3 on the same random-code operands and timing method as bench.py, so the
tcgen05 kernel's TFLOP/s can be put beside the library's on this box (power
cap included)."""
import sys, time
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev, generator=g).view(torch.float4_e2m1fn_x2)
b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device=dev, generator=g).view(torch.float4_e2m1fn_x2)
# scales: one e4m3 per 16 elements, swizzled 128x4 blocks (same tiling as our scales_tc)
sa = (torch.rand(n * n // 16, device=dev, generator=g) + 0.5).to(torch.float8_e4m3fn)
sb = (torch.rand(n * n // 16, device=dev, generator=g) + 0.5).to(torch.float8_e4m3fn)
try:
    out = torch._scaled_mm(a, b.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
except Exception as e:
    print("torch._scaled_mm NVFP4 unavailable:", repr(e)[:300])
    sys.exit(0)
torch.cuda.synchronize()
for _ in range(3):
    torch._scaled_mm(a, b.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
reps = 10
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
torch.cuda._sleep(1_000_000)
s.record()
for _ in range(reps):
    torch._scaled_mm(a, b.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(f"torch._scaled_mm NVFP4 {n}^3 bf16 out: {ms*1e3:.1f} us  {2*n**3/ms/1e9:.0f} TFLOP/s")
