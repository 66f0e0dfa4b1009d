"""Time K3 (dequantize) of a 65536x4096 container to bf16 / f32, L2 flushed,
next to write-bandwidth calibration (fill_ and a u8->bf16 copy).
Usage: [F46_DQ_VEC=1] python tools/time_dequant.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2512_02010_b200 import _lib
from paper_2512_02010_b200.blockquant import scales_tc_bytes

rows, cols = 65536, 4096
L = _lib.load()
if os.environ.get("F46_DQ_VEC"):  # tool-side switch onto the library test hook
    L.f46_set_test_hook(1, 1)
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(5)
codes = torch.randint(0, 256, (rows, cols // 2), generator=g, device=dev, dtype=torch.uint8)
scales = torch.randint(0, 0x7E, (scales_tc_bytes(rows, cols),), generator=g, device=dev, dtype=torch.uint8)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_r = torch.ones(128 << 20, dtype=torch.float16, device=dev)  # read sweep: leaves L2 clean
s = torch.cuda.current_stream().cuda_stream


def timed(fn, n=15):
    ts = []
    for i in range(n):
        flush.fill_(i)
        sink = torch.amax(flush_r)
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


tag = "vec" if os.environ.get("F46_DQ_VEC") else "tma"
for av in (float(np.float32(0.003)), 0.003):
    alpha = torch.tensor([av], dtype=torch.float64, device=dev)
    for od, dtc, ob in ((torch.bfloat16, _lib.DT_BF16, 2), (torch.float32, _lib.DT_F32, 4)):
        out = torch.empty((rows, cols), dtype=od, device=dev)
        ms = timed(lambda: L.f46_dequantize(codes.data_ptr(), scales.data_ptr(), 0, alpha.data_ptr(),
                                            rows, cols, out.data_ptr(), dtc, None, s))
        kind = "f32-alpha" if av == float(np.float32(av)) else "f64-alpha"
        print(f"K3[{tag}] {kind} -> {od}: {ms*1e3:.1f} us  {rows*cols*(0.5625+ob)/ms/1e6:.0f} GB/s")
big = torch.empty(rows * cols, dtype=torch.bfloat16, device=dev)
ms = timed(lambda: big.fill_(1.0))
print(f"calib fill_ bf16 {big.numel()*2/1e6:.0f} MB: {ms*1e3:.1f} us {big.numel()*2/ms/1e6:.0f} GB/s")
src = codes.view(-1)
dst = torch.empty(src.numel(), dtype=torch.bfloat16, device=dev)
ms = timed(lambda: dst.copy_(src))
print(f"calib u8->bf16 copy: {ms*1e3:.1f} us {src.numel()*3/ms/1e6:.0f} GB/s")
