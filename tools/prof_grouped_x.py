import sys, torch
sys.path.insert(0, ".")
import bench, paper_2512_02010_b200 as f46
dev = torch.device("cuda", 0)
t = bench.moe_tensors(dev)
cfg = f46.QuantConfig(scale_mode="adaptive")
for i in range(3):
    f46.quantize_grouped(t["x"], cfg, check_finite=False)
torch.cuda.synchronize()
