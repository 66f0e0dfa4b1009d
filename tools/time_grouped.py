"""Time the grouped MoE quantizers on bench.moe_tensors (L2 flushed, CUDA events)
and print per-expert alpha / tie direction of the 1-D operands."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2512_02010_b200 as f46
dev = torch.device("cuda", 0)
t = bench.moe_tensors(dev)
cfg = f46.QuantConfig(scale_mode="adaptive")
flush = bench.L2Flush(dev)
s = torch.cuda.current_stream()
for name in ("x", "h", "dy", "dh"):
    ms = bench.timed_flushed(lambda: f46.quantize_grouped(t[name], cfg, check_finite=False), flush, s, 10)
    q = f46.quantize_grouped(t[name], cfg)
    am = t[name].float().abs().amax(dim=(1, 2))
    al = (am / 1536.0).float()
    td = ["0" if float(a) * 1536 == float(m) else ("-" if float(a) * 1536 > float(m) else "+") for a, m in zip(al, am)]
    print(f"{name} {tuple(t[name].shape)}: {ms*1e3:.1f} us  {t[name].numel()*4.5625/ms/1e6:.0f} GB/s  tdir {''.join(td)}")
# per expert (single-tensor calls): which experts are slow
for e in range(t["x"].shape[0]):
    xe = t["x"][e]
    ms = bench.timed_flushed(lambda: f46.quantize_tensor_adaptive(xe, cfg, check_finite=False), flush, s, 5)
    am = float(xe.float().abs().max())
    a = float(torch.tensor(am / 1536.0, dtype=torch.float32))
    sig = int(torch.tensor([a], dtype=torch.float32).view(torch.int32).item()) & 0x7FFFFF | 0x800000
    while sig % 2 == 0:
        sig //= 2
    print(f"  x[{e}] amax {am} alpha {a:.9g} odd(alpha) {sig}: {ms*1e3:.1f} us")
