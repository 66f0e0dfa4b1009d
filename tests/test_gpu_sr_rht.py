"""GPU parity of the gradient recipe: stochastic rounding with the reference's
exact Philox uniforms (f46_quantize_sr; blockquant.py:253-257,
codecs.py:120-148), the 16-wide randomized Hadamard transform (f46_rht16;
transforms.py:92-105), and linear_dgrad / linear_wgrad with rounding='sr'
(qlinear.py:123-159).  Quantization and the transform are bit-exact against
reference fixtures (tests/golden/golden_sr.npz); the GEMM outputs meet the
reference's matmul bound (relative Frobenius <= 1e-5).
"""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from tests.golden_util import load

pytestmark = pytest.mark.gpu

CASES = load("golden_sr.npz")


def to_torch(x):
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


SR = [c for c in CASES if c[0].startswith("sr_")]
RHT = [c for c in CASES if c[0].startswith("rht_")]
GRAD = [c for c in CASES if c[0].startswith("grad_")]


@pytest.mark.parametrize("name,rec", SR, ids=[c[0] for c in SR])
def test_stochastic_rounding_bit_exact(name, rec):
    mode = str(rec["mode"])
    cfg = f46.QuantConfig(scale_mode=mode, rounding="sr", seed=int(rec["seed"]))
    fn = f46.quantize_tensor_adaptive if mode == "adaptive" else f46.quantize_tensor
    q = fn(to_torch(rec["x"]), cfg, sr_tag=int(rec["tag"]), want_rowmajor=True)
    assert q.alpha == float(rec["alpha"])
    assert np.array_equal(q.scales_rm.cpu().numpy(), rec["scales"])
    assert np.array_equal(q.packed_codes.cpu().numpy(), rec["codes"])


@pytest.mark.parametrize("name,rec", RHT, ids=[c[0] for c in RHT])
def test_rht_bit_exact(name, rec):
    spec = f46.RhtSpec(seed=int(rec["seed"]))
    x = torch.from_numpy(rec["x"]).cuda()
    assert torch.equal(f46.apply_rht(x, spec).cpu(), torch.from_numpy(rec["y"]))
    assert torch.equal(f46.invert_rht(x, spec).cpu(), torch.from_numpy(rec["inv"]))


def rel_fro(got, ref):
    got, ref = got.double(), ref.double()
    return float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))


@pytest.mark.parametrize("name,rec", GRAD, ids=[c[0] for c in GRAD])
def test_sr_gradient_recipes_match_reference(name, rec):
    cfg = f46.QuantConfig(scale_mode=str(rec["mode"]), rounding="sr", seed=3)
    dx = f46.linear_dgrad(to_torch(rec["dy"]), to_torch(rec["W"]), cfg)
    dw = f46.linear_wgrad(to_torch(rec["dy"]), to_torch(rec["x"]), cfg)
    assert rel_fro(dx, torch.from_numpy(rec["dx"]).cuda()) <= 1e-5
    assert rel_fro(dw, torch.from_numpy(rec["dw"]).cuda()) <= 1e-5


def test_sr_is_unbiased_in_expectation():
    """Mean of SR dequantizations over many seeds approaches the input
    (the reference's statistical SR property, test_qlinear.py)."""
    g = torch.Generator().manual_seed(9)
    x = torch.randn(64, 64, generator=g).to(torch.bfloat16).cuda()
    acc = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    n = 64
    for s in range(n):
        cfg = f46.QuantConfig(scale_mode="fixed6", rounding="sr", seed=s)
        acc += f46.dequantize_tensor(f46.quantize_tensor(x, cfg), torch.float64)
    err_sr = float((acc / n - x.double()).abs().mean())
    err_rne = float((f46.dequantize_tensor(f46.quantize_tensor(x, f46.QuantConfig()), torch.float64)
                     - x.double()).abs().mean())
    assert err_sr < 0.5 * err_rne


@pytest.mark.parametrize("mode", ["adaptive", "fixed6"])
def test_sr_fast_path_matches_float64_path(mode):
    """BF16 input takes the f32-bracket SR path (sr_code_fast, float64 only
    near a decision boundary); the same values as float64 input take the
    float64 restatement everywhere.  2M elements, every code and scale equal."""
    g = torch.Generator().manual_seed(17)
    x = torch.randn(512, 4096, generator=g).to(torch.bfloat16)
    cfg = f46.QuantConfig(scale_mode=mode, rounding="sr", seed=9)
    fn = f46.quantize_tensor_adaptive if mode == "adaptive" else f46.quantize_tensor
    a = fn(x.cuda(), cfg, sr_tag=1)
    b = fn(x.double().cuda(), cfg, sr_tag=1)
    assert a.alpha == b.alpha
    assert torch.equal(a.scales_tc, b.scales_tc)
    assert torch.equal(a.packed_codes, b.packed_codes)


def test_rht_bf16_vector_path_matches_float64_input():
    """The BF16 kernel (16-byte loads / stores) and the float64-input kernel
    compute the same float64 butterflies: identical outputs, also unaligned."""
    g = torch.Generator().manual_seed(4)
    x = torch.randn(256, 1024, generator=g).to(torch.bfloat16).cuda()
    spec = f46.RhtSpec(seed=6)
    a = f46.apply_rht(x, spec)
    b = f46.apply_rht(x.double(), spec)
    assert torch.equal(a, b)
    xs = x.reshape(-1)[16:16 + 4096]  # 32-byte offset view: still 16-byte aligned
    assert torch.equal(f46.apply_rht(xs, spec), f46.apply_rht(xs.double(), spec))
