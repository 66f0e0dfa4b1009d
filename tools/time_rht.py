"""Time the WGRAD-operand kernels (transpose + RHT16, amax pass and quantize
pass) on the config-5 activation/gradient shapes, L2 flushed before each run.
Usage: [F46_LIB_PATH=..] python tools/time_rht.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
from paper_2512_02010_b200 import _lib
from paper_2512_02010_b200.grouped import sign_mask, _empty, _stream, _DT_OF
DT = _DT_OF[torch.bfloat16]

dev = torch.device("cuda")
E, T = 16, 3072
L = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
spec = f46.RhtSpec(seed=0)
mask = sign_mask(spec)


def timed(fn, n=10):
    ts = []
    for _ in range(n + 3):
        flush.fill_(1)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts = sorted(ts[3:])
    return ts[len(ts) // 2]


for name, H, std in (("x", 2688, 1.0), ("dy", 2688, 1e-3), ("h", 1856, 1.0)):
    g = torch.Generator(device=dev).manual_seed(5)
    t = (torch.randn(E, T, H, generator=g, device=dev) * std).to(torch.bfloat16)
    amax = torch.zeros(E, dtype=torch.float64, device=dev)
    codes, scales = _empty(E, H, T, dev, zero_scales=True)
    alpha = torch.empty(E, dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    st = _stream()
    fa = lambda: L.f46_rht_t_amax_grouped(t.data_ptr(), DT, E, T, H, mask, amax.data_ptr(), st)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    from paper_2512_02010_b200.grouped import _mcap
    mc = _mcap(cfg)
    fq = lambda: L.f46_quantize_rht_t_grouped(t.data_ptr(), DT, E, T, H, mask, _lib.MODE["adaptive"], _lib.RULE["mse"],
                                              mc, amax.data_ptr(), codes.data_ptr(), scales.data_ptr(),
                                              alpha.data_ptr(), flags.data_ptr(), st)
    amax.zero_(); fa()
    ua, uq = timed(fa), timed(fq)
    n = E * T * H
    print(f"{name} [{E},{T},{H}] amax {ua:7.1f} us {2 * n / ua / 1e3:6.0f} GB/s | quant {uq:7.1f} us "
          f"{2.5625 * n / uq / 1e3:6.0f} GB/s | both {(ua + uq):7.1f} us")
