"""Config 1 (4096^2 N(0,1) BF16): fixed6 vs adaptive through bench.bench_c1."""
import sys, torch
sys.path.insert(0, ".")
import bench
class A: steps = 10
peaks, _ = bench.measured_peaks()
r = bench.bench_c1(A(), torch.device("cuda", 0), peaks)
print(f"c1 fixed6 {r['fixed6']['ms'] * 1e3:.1f} us (k2 {r['fixed6']['k2_ms'] * 1e3:.1f}) adaptive "
      f"{r['adaptive']['ms'] * 1e3:.1f} us (k2 {r['adaptive']['k2_ms'] * 1e3:.1f}) overhead "
      f"{r['overhead_end_to_end']:.3f} k2 {r['overhead_k2']:.3f}")
