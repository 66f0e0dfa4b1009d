"""quantize_weights_2d on a 4096x14336 BF16 weight a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(11)
W = (torch.randn(4096, 14336, generator=g, device=dev) * 0.02).to(torch.bfloat16)
cfg = f46.QuantConfig(scale_mode="adaptive")
for _ in range(3):
    f46.quantize_weights_2d(W, cfg, check_finite=False)
torch.cuda.synchronize()
