"""GPU parity of the 2-D 16x16-tile weight quantizer (f46_quantize_2d,
reference transforms.py:134-179) and of the linear-layer recipes built on it
(qlinear.py:107-135: FPROP x @ W^T and DGRAD dy @ W on tcgen05).

Tile quantization is bit-exact against the reference's own fixtures
(tests/golden/golden_tile2d.npz) and against the CPU oracle on ragged shapes;
the transposed container is checked to be the exact transpose; the linear
outputs are checked against the reference's linear_forward / linear_dgrad
(tests/golden/golden_linear.npz) to the reference's matmul bound, relative
Frobenius <= 1e-5.
"""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from oracle import oracle as O
from tests.golden_util import load

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5


def to_torch(x: np.ndarray) -> torch.Tensor:
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


TILES = load("golden_tile2d.npz")


@pytest.mark.parametrize("name,rec", TILES, ids=[c[0] for c in TILES])
def test_tile2d_golden(name, rec):
    q = f46.quantize_weights_2d(to_torch(rec["x"]), f46.QuantConfig(scale_mode=str(rec["mode"])),
                                want_rowmajor=True)
    assert q.alpha == float(rec["alpha"])
    assert np.array_equal(q.scales_rm.cpu().numpy(), rec["scales"])
    assert np.array_equal(q.packed_codes.cpu().numpy(), rec["codes"])


def bf16_bits(shape, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    x = (torch.randn(*shape, generator=g) * std).to(torch.bfloat16)
    return x, x.view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
@pytest.mark.parametrize("shape", [(64, 96), (40, 50), (33, 17), (256, 1024), (1856, 2688)])
def test_tile2d_matches_oracle(mode, shape):
    x, bits = bf16_bits(shape, sum(shape), std=0.03)
    q = f46.quantize_weights_2d(x.cuda(), f46.QuantConfig(scale_mode=mode), want_rowmajor=True)
    ref = O.quantize_2d(bits, mode)
    assert q.alpha == ref["alpha"]
    assert np.array_equal(q.scales_rm.cpu().numpy(), ref["scales"])
    assert np.array_equal(q.packed_codes.cpu().numpy(), ref["codes"])


@pytest.mark.parametrize("shape", [(48, 32), (40, 50), (300, 200)])
def test_transposed_container_is_exact_transpose(shape):
    x, _ = bf16_bits(shape, 7)
    q = f46.quantize_weights_2d(x.cuda(), f46.QuantConfig(scale_mode="adaptive"))
    d = f46.dequantize_tensor(q, torch.float64)
    dt = f46.dequantize_tensor(q.transposed, torch.float64)
    assert q.transposed.shape == (shape[1], shape[0])
    assert torch.equal(dt, d.T)


def rel_fro(got, ref):
    got, ref = got.double(), ref.double()
    return float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))


LINEAR = load("golden_linear.npz")


@pytest.mark.parametrize("name,rec", LINEAR, ids=[c[0] for c in LINEAR])
def test_linear_forward_dgrad_match_reference(name, rec):
    cfg = f46.QuantConfig(scale_mode=str(rec["mode"]))
    y = f46.linear_forward(to_torch(rec["x"]), to_torch(rec["W"]), cfg)
    dx = f46.linear_dgrad(to_torch(rec["dy"]), to_torch(rec["W"]), cfg)
    assert rel_fro(y, torch.from_numpy(rec["y"]).cuda()) <= REL_TOL
    assert rel_fro(dx, torch.from_numpy(rec["dx"]).cuda()) <= REL_TOL


def test_dgrad_gemm_is_tensor_core_transpose_product():
    """dy @ W through W^T's container equals the f64 product of the exact
    dequantized operands (MoE expert shape: out 1856, in 2688)."""
    x, _ = bf16_bits((1856, 2688), 3, std=0.02)
    dy, _ = bf16_bits((512, 1856), 4)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    dx = f46.linear_dgrad(dy.cuda(), x.cuda(), cfg)
    dyq = f46.quantize_tensor_adaptive(dy.cuda(), cfg)
    wq = f46.quantize_weights_2d(x.cuda(), cfg)
    ref = f46.dequantize_tensor(dyq, torch.float64) @ f46.dequantize_tensor(wq, torch.float64)
    assert rel_fro(dx, ref) <= REL_TOL
