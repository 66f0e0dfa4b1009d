"""Run the hot kernels a few times on the c3 tensor (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
from paper_2512_02010_b200 import _lib
from paper_2512_02010_b200.blockquant import scales_tc_bytes

rows, cols = int(os.environ.get("ROWS", 65536)), int(os.environ.get("COLS", 4096))
mode = os.environ.get("MODE", "adaptive")
dt = os.environ.get("DT", "bf16")
L = _lib.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(int(os.environ.get("SEED", 1234)))
x = torch.randn(rows, cols, generator=g, device=dev)
x = x.to(torch.bfloat16) if dt == "bf16" else x
codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device=dev)
scales = torch.empty(scales_tc_bytes(rows, cols), dtype=torch.uint8, device=dev)
amax = torch.zeros(1, dtype=torch.float64, device=dev)
s = torch.cuda.current_stream().cuda_stream
DT = _lib.DT_BF16 if dt == "bf16" else _lib.DT_F32
mcap = {"adaptive": 1536.0, "fixed6": 2688.0, "fixed4": 1792.0}[mode]
for i in range(int(os.environ.get("ITERS", 3))):
    amax.zero_()
    L.f46_amax(x.data_ptr(), DT, x.numel(), amax.data_ptr(), s)
    L.f46_quantize(x.data_ptr(), DT, rows, cols, _lib.MODE[mode], 0, mcap, amax.data_ptr(), 0.0,
                   codes.data_ptr(), scales.data_ptr(), None, None, None, None, s)
    if os.environ.get("DEQ"):
        out = torch.empty((rows, cols), dtype=torch.bfloat16, device=dev)
        alpha = torch.tensor([float(torch.tensor(0.003, dtype=torch.float32))], dtype=torch.float64, device=dev)  # f32-exact, as quantize writes it
        L.f46_dequantize(codes.data_ptr(), scales.data_ptr(), 0, alpha.data_ptr(), rows, cols,
                         out.data_ptr(), _lib.DT_BF16, None, s)
torch.cuda.synchronize()
print("done")
