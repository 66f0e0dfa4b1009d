import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2512_02010_b200 as f46
dev = torch.device("cuda", 0)
t = bench.moe_tensors(dev)
cfg = f46.QuantConfig(scale_mode="adaptive")
bench.moe_step(t, cfg)
torch.cuda.synchronize()
bench.moe_step(t, cfg)
torch.cuda.synchronize()
