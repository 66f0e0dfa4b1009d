"""Time SR 4/6 quantization (amax + quant_sr4_kernel) of a 16384x4096 BF16 tensor, L2 flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2512_02010_b200 as f46
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(11)
X = torch.randn(16384, 4096, generator=g, device=dev).to(torch.bfloat16)
sr = f46.QuantConfig(scale_mode="adaptive", rounding="sr", seed=3)
flush = bench.L2Flush(dev)
ms = bench.timed_flushed(lambda: f46.quantize_tensor_adaptive(X, sr, sr_tag=2, check_finite=False), flush,
                         torch.cuda.current_stream(), 5)
print(f"{os.path.basename(os.environ.get('F46_LIB_PATH', 'default'))} SR 16384x4096: {ms * 1e3:.1f} us")
