"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): K1 amax, K2 quantize (streaming whole-
segment and ragged paths, BF16 and FP32), K3 dequantize (TMA and coalesced),
K4 tcgen05 GEMM (CTA pair, grouped, fused amax), 2-D tiles, SR, RHT, stats,
grouped MoE quantizers and the block-level kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2512_02010_b200 as f46
from paper_2512_02010_b200 import _lib

torch.manual_seed(0)
dev = torch.device("cuda")
cfg = f46.QuantConfig(scale_mode="adaptive")
for shape in ((256, 4096), (130, 2688), (33, 48)):
    x = torch.randn(*shape, device=dev).to(torch.bfloat16)
    q = f46.quantize_tensor_adaptive(x, cfg)
    f46.quantize_tensor(x.float(), f46.QuantConfig(), )
    for dt in (torch.float64, torch.float32, torch.bfloat16):
        f46.dequantize_tensor(q, dt)
a = f46.quantize_tensor_adaptive(torch.randn(512, 1024, device=dev).to(torch.bfloat16), cfg)
b = f46.quantize_tensor_adaptive(torch.randn(384, 1024, device=dev).to(torch.bfloat16), cfg)
f46.gemm_nvfp4(a, b, torch.bfloat16)
f46.gemm_nvfp4(a, b, torch.float32, amax_out=torch.zeros(1, dtype=torch.float64, device=dev))
X = torch.randn(2, 256, 512, device=dev).to(torch.bfloat16)
g = f46.quantize_grouped(X, cfg)
W = (torch.randn(2, 192, 512, device=dev) * 0.02).to(torch.bfloat16)
gw = f46.quantize_weights_2d_grouped(W, cfg)
f46.gemm_nvfp4_grouped(*g.operands(), *gw.operands(), 256, 192, 512, torch.bfloat16)
gr = f46.quantize_wgrad_operand_grouped(X, cfg)
f46.quantize_weights_2d(W[0], cfg)
f46.quantize_tensor_adaptive(torch.randn(64, 256, device=dev), f46.QuantConfig(scale_mode="adaptive", rounding="sr", seed=1))
f46.apply_rht(torch.randn(64, 64, device=dev), f46.RhtSpec(seed=0))
f46.selection_stats(torch.randn(128, 256, device=dev), cfg)
f46.quantize_block(torch.randn(37).numpy(), 0.01, 6.0)
f46.emulated_fp4_matmul(f46.quantize_tensor_adaptive(torch.randn(40, 64, device=dev), cfg),
                        f46.quantize_tensor_adaptive(torch.randn(64, 48, device=dev), cfg))
# K2 through the two-kernel path (parallel-resolver instantiation) on a tensor
# whose tie direction is +1 (collapsed scale brackets), and a chunked launch
from paper_2512_02010_b200.sharded import ShardedQuantizer
xs = torch.randn(256, 4096, device=dev).to(torch.bfloat16)
xs[3, 5] = 7.0
sq = ShardedQuantizer(256, 4096, torch.bfloat16, dev, "adaptive", all_reduce_max=lambda t: None)
sq(xs)
_lib.load().f46_set_test_hook(_lib.HOOK["seg_chunk_bytes"], 128 * 4096 * 2)
sq.amax_local(xs, torch.cuda.current_stream().cuda_stream)
sq.quantize_local(xs, torch.cuda.current_stream().cuda_stream)
_lib.load().f46_set_test_hook(_lib.HOOK["seg_chunk_bytes"], 0)
torch.cuda.synchronize()
print("sanitize workload done")
