"""Time the grouped NVFP4 GEMM on the config-5 MoE expert shapes (16 experts,
3072 tokens each) with random codes/scales.  Usage: [F46_LIB_PATH=..] python tools/time_moe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
from paper_2512_02010_b200.blockquant import scales_tc_bytes

dev = torch.device("cuda")
E, T, H, F = 16, 3072, 2688, 1856
g = torch.Generator(device=dev).manual_seed(0)


def operand(rows, k):
    nb = -(-k // 16)
    nbp = nb + (nb & 1)
    codes = torch.randint(0, 256, (E, rows, nbp * 8), generator=g, device=dev, dtype=torch.uint8)
    sc = torch.randint(0x30, 0x40, (E, scales_tc_bytes(rows, nbp * 16)), generator=g, device=dev,
                       dtype=torch.uint8)
    return codes, sc, torch.ones(E, dtype=torch.float64, device=dev), nbp * 16


shapes = {"fprop_x_w1": (T, F, H), "fprop_h_w2": (T, H, F), "wgrad_dh_x": (F, H, T)}
tot_f = tot_ms = 0.0
for name, (M, N, K) in shapes.items():
    a = operand(M, K)
    b = operand(N, K)
    Kp = a[3]
    run = lambda: f46.gemm_nvfp4_grouped(a[0], a[1], a[2], b[0], b[1], b[2], M, N, Kp, torch.bfloat16)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    fl = 2.0 * E * M * N * K
    tot_f += fl
    tot_ms += ms
    print(f"{name} M={M} N={N} K={K}: {ms*1e3:.1f} us {fl/ms/1e9:.0f} TFLOP/s")
print(f"total {tot_f/tot_ms/1e9:.0f} TFLOP/s")
