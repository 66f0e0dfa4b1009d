import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2512_02010_b200 import _lib
L = _lib.load()
class A: steps = 10
peaks, _ = bench.measured_peaks()
r = bench.bench_weights(A(), L, torch.device("cuda", 0), peaks)
print({k: (round(v["ms"] * 1e3, 1), round(v["frac_of_hbm"], 3)) for k, v in r.items()})
