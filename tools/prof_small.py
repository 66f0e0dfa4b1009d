"""Config-2 weight quantize through ShardedQuantizer (world 1: the fused
amax + quantize launch), a few calls, for an ncu launch list / capture."""
import sys, torch
sys.path.insert(0, ".")
from paper_2512_02010_b200.sharded import ShardedQuantizer
dev = torch.device("cuda", 0)
r, c = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 4096)))
w = (torch.randn(r, c, device=dev) * 0.02).to(torch.bfloat16)
sq = ShardedQuantizer(r, c, torch.bfloat16, dev, "adaptive")
for _ in range(4):
    sq(w)
torch.cuda.synchronize()
