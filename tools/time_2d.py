"""Time quantize_weights_2d (amax + 2-D tiles, W and W^T) on a 4096x14336 BF16 weight."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2512_02010_b200 as f46
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(11)
W = (torch.randn(4096, 14336, generator=g, device=dev) * 0.02).to(torch.bfloat16)
cfg = f46.QuantConfig(scale_mode="adaptive")
flush = bench.L2Flush(dev)
ms = bench.timed_flushed(lambda: f46.quantize_weights_2d(W, cfg, check_finite=False), flush,
                         torch.cuda.current_stream(), 10)
by = W.numel() * (2 * 2 + 2 * 0.5625)
print(f"{os.path.basename(os.environ.get('F46_LIB_PATH', 'default'))} 2-D 4096x14336: {ms*1e3:.1f} us {by/ms/1e6:.0f} GB/s")
