"""Fused amax + quantize (ShardedQuantizer, one rank) at 4096 columns and several row counts."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2512_02010_b200.sharded import ShardedQuantizer
dev = torch.device("cuda", 0)
flush = bench.L2Flush(dev)
s = torch.cuda.current_stream()
for r in (4096, 6144, 8192, 12288):
    g = torch.Generator(device=dev).manual_seed(r)
    w = (torch.randn(r, 4096, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    am = float(w.float().abs().max())
    sq = ShardedQuantizer(r, 4096, torch.bfloat16, dev, "adaptive")
    ms = bench.timed_flushed(lambda: sq(w), flush, s, 10, warm=3)
    print(f"fused {r}x4096: {ms * 1e3:.1f} us  {w.numel() * 4.5625 / ms / 1e6:.0f} GB/s  fused={sq.fused} amax {am}")
