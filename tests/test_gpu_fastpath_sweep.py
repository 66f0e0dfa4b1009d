"""Fast paths vs the float64 restatement on random shapes.

Every quantizer family has an f32 fast path (bracketed codes and scales,
certified decisions) for BF16/F32 input and the float64 line-by-line
restatement of the reference for float64 input.  Feeding the same values both
ways must give identical containers; ragged shapes, tiny rows, odd block
counts and a spread of magnitudes exercise tails, padding and the deferred
/ fallback branches."""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46

pytestmark = pytest.mark.gpu

SHAPES = [(1, 16), (3, 48), (7, 100), (33, 80), (130, 272), (257, 64), (64, 1040), (5, 4112),
          (200, 2048), (1, 4096)]
SCALES = [1.0, 3e-3, 250.0]


def values(shape, seed, scale):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(*shape, generator=g) * scale
    # heavy tails and exact zeros inside blocks
    x[..., ::7] *= 8.0
    x[..., 3::11] = 0.0
    return x.to(torch.bfloat16)


def same(a, b):
    assert a.alpha == b.alpha
    assert torch.equal(a.scales_tc, b.scales_tc)
    assert torch.equal(a.packed_codes, b.packed_codes)


@pytest.mark.parametrize("scale", SCALES)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
def test_quantize_fast_equals_float64(shape, mode, scale):
    x = values(shape, shape[0] * 131 + shape[1], scale)
    cfg = f46.QuantConfig(scale_mode=mode)
    fn = f46.quantize_tensor_adaptive if mode == "adaptive" else f46.quantize_tensor
    same(fn(x.cuda(), cfg), fn(x.double().cuda(), cfg))
    same(fn(x.float().cuda(), cfg), fn(x.double().cuda(), cfg))


@pytest.mark.parametrize("shape", SHAPES)
def test_sr_fast_equals_float64(shape):
    x = values(shape, shape[0] + 7 * shape[1], 1.0)
    cfg = f46.QuantConfig(scale_mode="adaptive", rounding="sr", seed=5)
    same(f46.quantize_tensor_adaptive(x.cuda(), cfg, sr_tag=3),
         f46.quantize_tensor_adaptive(x.double().cuda(), cfg, sr_tag=3))


@pytest.mark.parametrize("shape", [(16, 16), (40, 50), (33, 17), (130, 272), (64, 1040)])
@pytest.mark.parametrize("mode", ["adaptive", "fixed6"])
def test_tile2d_fast_equals_float64(shape, mode):
    x = values(shape, 3 * shape[0] + shape[1], 0.02)
    cfg = f46.QuantConfig(scale_mode=mode)
    a = f46.quantize_weights_2d(x.cuda(), cfg)
    b = f46.quantize_weights_2d(x.double().cuda(), cfg)
    same(a, b)
    same(a.transposed, b.transposed)


@pytest.mark.parametrize("shape", SHAPES[3:])
def test_stats_fast_equals_float64(shape):
    x = values(shape, 11 * shape[0] + shape[1], 1.0)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    a = f46.selection_stats(x.cuda(), cfg)
    b = f46.selection_stats(x.double().cuda(), cfg)
    assert a.fraction_4 == b.fraction_4 and a.disagreements == b.disagreements
    assert a.aggregate_mse == b.aggregate_mse


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_dequant_routes_agree(shape, dtype):
    x = values(shape, shape[0] * 17 + shape[1], 1.0)
    q = f46.quantize_tensor_adaptive(x.cuda(), f46.QuantConfig(scale_mode="adaptive"))
    d64 = f46.dequantize_tensor(q, torch.float64).cpu().numpy()
    d = f46.dequantize_tensor(q, dtype).cpu()
    if dtype == torch.float32:
        assert np.array_equal(d.numpy(), d64.astype(np.float32))
    else:
        # one rounding of the float64 value (torch's f64 -> bf16 goes through f32)
        from tests.test_gpu_quant import f64_to_bf16_bits
        assert np.array_equal(d.view(torch.int16).numpy().view(np.uint16), f64_to_bf16_bits(d64))


@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
def test_tile2d_v2_special_tiles_equal_v1(mode, test_hook):
    """The two-tiles-per-warp 2-D kernel against the one-tile-per-warp kernel
    on all-zero tiles (with -0.0), tiles beyond the fast path's magnitude
    range (float32 input, 1e30) and ragged edges."""
    g = torch.Generator().manual_seed(8)
    x = torch.randn(70, 90, generator=g) * 0.02
    x[:16, :16] = 0.0
    x[0:16:3, 0:16:5] = -0.0
    x[16:32, 32:48] *= 1e32          # tile max ~1e30: float64 tile path
    x[48:64, 16:32] = 1e-30          # tiny tile
    for t in (x.float(), x.to(torch.bfloat16)):
        cfg = f46.QuantConfig(scale_mode=mode)
        a = f46.quantize_weights_2d(t.cuda(), cfg, want_rowmajor=True)
        test_hook("q2_v1", 1)
        b = f46.quantize_weights_2d(t.cuda(), cfg, want_rowmajor=True)
        test_hook("q2_v1", 0)
        same(a, b)
        same(a.transposed, b.transposed)
        assert torch.equal(a.scales_rm, b.scales_rm)
