"""Time K2 (fused quantize) and K1 (amax) on the c3 tensor with CUDA events.
Usage: F46_LIB_PATH=... python tools/time_quant.py [mode] [dtype]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_02010_b200 import _lib
from paper_2512_02010_b200.blockquant import scales_tc_bytes

mode = sys.argv[1] if len(sys.argv) > 1 else "adaptive"
dt = sys.argv[2] if len(sys.argv) > 2 else "bf16"
rows, cols = int(os.environ.get("ROWS", 65536)), int(os.environ.get("COLS", 4096))
L = _lib.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(int(os.environ.get("SEED", 1234)))
x = torch.randn(rows, cols, generator=g, device=dev) * float(os.environ.get("STD", 1.0))
if os.environ.get("AMAX"):  # pin the tensor's amax (its tie direction): values scaled below it
    x = x * (float(os.environ["AMAX"]) / (x.abs().max() * 1.001))
    x.view(-1)[12345] = float(os.environ["AMAX"])
x = x.to(torch.bfloat16) if dt == "bf16" else x
DT = _lib.DT_BF16 if dt == "bf16" else _lib.DT_F32
codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device=dev)
scales = torch.empty(scales_tc_bytes(rows, cols), dtype=torch.uint8, device=dev)
amax = torch.zeros(1, dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_r = torch.ones(128 << 20, dtype=torch.float16, device=dev)  # read sweep: leaves L2 clean
s = torch.cuda.current_stream().cuda_stream
mcap = {"adaptive": 1536.0, "fixed6": 2688.0, "fixed4": 1792.0}[mode]
L.f46_amax(x.data_ptr(), DT, x.numel(), amax.data_ptr(), s)
ts = []
for i in range(25):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(i)
        sink = torch.amax(flush_r)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.f46_quantize(x.data_ptr(), DT, rows, cols, _lib.MODE[mode], 0, mcap, amax.data_ptr(), 0.0,
                   codes.data_ptr(), scales.data_ptr(), None, None, None, None, s)
    b.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b))
ms = sum(ts) / len(ts)
bpe = (2 if dt == "bf16" else 4) + 0.5625
ta = []
for i in range(25):
    flush.fill_(i)
    sink = torch.amax(flush_r)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.f46_amax(x.data_ptr(), DT, x.numel(), amax.data_ptr(), s)
    b.record()
    torch.cuda.synchronize()
    if i >= 5:
        ta.append(a.elapsed_time(b))
ma = sum(ta) / len(ta)
am = float(amax.item())
al = float(torch.tensor(am, dtype=torch.float32) / torch.tensor(mcap, dtype=torch.float32))
tdir = "-1" if al * mcap > am else ("+1" if al * mcap < am else "0")
print(f"seed {os.environ.get('SEED', 1234)} amax {am} alpha {al} tdir {tdir} ", end="")
print(f"{os.path.basename(os.environ.get('F46_LIB_PATH', 'default'))} {mode} {dt}: K2 {ms*1e3:.1f} us  {rows*cols*bpe/ms/1e6:.0f} GB/s | K1 amax {ma*1e3:.1f} us {rows*cols*(bpe-0.5625)/ma/1e6:.0f} GB/s")
if os.environ.get("NODQ"):
    sys.exit(0)
# K3 dequantize of the same tensor (bf16 and f32 out)
alpha = torch.tensor([0.003], dtype=torch.float64, device=dev)
for od, dtc, ob in ((torch.bfloat16, _lib.DT_BF16, 2), (torch.float32, _lib.DT_F32, 4)):
    out = torch.empty((rows, cols), dtype=od, device=dev)
    td = []
    for i in range(15):
        flush.fill_(i)
        sink = torch.amax(flush_r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.f46_dequantize(codes.data_ptr(), scales.data_ptr(), 0, alpha.data_ptr(), rows, cols,
                         out.data_ptr(), dtc, None, s)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            td.append(a.elapsed_time(b))
    md = sum(td) / len(td)
    print(f"  K3 dequant -> {od}: {md*1e3:.1f} us  {rows*cols*(0.5625+ob)/md/1e6:.0f} GB/s")
