import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
g = torch.Generator(device="cuda").manual_seed(11)
X = torch.randn(16384, 4096, generator=g, device="cuda").to(torch.bfloat16)
sr = f46.QuantConfig(scale_mode="adaptive", rounding="sr", seed=3)
for _ in range(2):
    f46.quantize_tensor_adaptive(X, sr, sr_tag=2, check_finite=False)
torch.cuda.synchronize()
