"""Print the blocks where the GPU quantizer differs from the golden fixture."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_02010_b200 as f46
from tests.golden_util import quant_cases, opt
from oracle import oracle as O
name = sys.argv[1]
rec = dict(quant_cases())[name]
x = rec["x"]; cols = x.shape[-1]; rows = x.size // cols
xt = torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda() if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
mode = str(rec["mode"])
cfg = f46.QuantConfig(scale_mode=mode)
q = (f46.quantize_tensor_adaptive if mode == "adaptive" else f46.quantize_tensor)(xt, cfg, alpha=opt(rec["alpha_override"]), want_rowmajor=True, want_pick4=True)
print("alpha", q.alpha, rec["alpha"])
gc = q.packed_codes.cpu().numpy().reshape(rows, -1); rc = rec["codes"].reshape(rows, -1)
gs = q.scales_rm.cpu().numpy(); rs = rec["scales"].reshape(rows, -1)
gp = q.pick4.cpu().numpy(); rp = rec["pick4"].reshape(rows, -1)
x64 = O.bf16_to_f64(x) if x.dtype == np.uint16 else x.astype(np.float64)
x64 = x64.reshape(rows, cols)
for r in range(rows):
    for b in range(gs.shape[1]):
        if (gc[r, 8*b:8*b+8] != rc[r, 8*b:8*b+8]).any() or gs[r, b] != rs[r, b] or gp[r, b] != rp[r, b]:
            print("row", r, "blk", b, "x", x64[r, 16*b:16*b+16].tolist())
            print("  gpu sc", gs[r, b], "pick4", gp[r, b], "codes", O.unpack_codes(gc[r:r+1, 8*b:8*b+8], 16).tolist())
            print("  ref sc", rs[r, b], "pick4", rp[r, b], "codes", O.unpack_codes(rc[r:r+1, 8*b:8*b+8], 16).tolist())
