"""Grouped (per-MoE-expert) quantization against the oracle, bit for bit.

Each expert is its own reference tensor with its own tensor scale
(blockquant.py:215-222), so every group must equal the oracle run on that
expert alone: packed codes, tcgen05 scales (read back row-major) and alpha.
The WGRAD operand (reference qlinear.py:150-157: apply_rht(a.T) then 1-D
quantization along tokens) is checked against oracle.apply_rht (pinned to the
reference's RHT fixture, tests/test_oracle_rht.py) followed by the oracle's
float64 quantizer.
"""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from oracle import oracle as O
from paper_2512_02010_b200.blockquant import tc_to_rowmajor

pytestmark = pytest.mark.gpu


def bf16_stack(E, shape, seed, stds):
    g = torch.Generator().manual_seed(seed)
    xs = [(torch.randn(*shape, generator=g) * s).to(torch.bfloat16) for s in stds[:E]]
    return torch.stack(xs)


def bits(x: torch.Tensor) -> np.ndarray:
    return x.contiguous().view(torch.int16).numpy().view(np.uint16)


def check_group(gq, e, ref, rows, cols):
    q = gq.group(e)
    assert float(q.alpha_dev.item()) == ref["alpha"], e
    got = q.packed_codes.cpu().numpy()
    bad = np.argwhere(got != ref["codes"])
    assert bad.size == 0, f"expert {e}: {len(bad)} code bytes differ, first {bad[:4].tolist()}"
    sc = tc_to_rowmajor(q.scales_tc, rows, -(-cols // 16)).cpu().numpy()
    assert np.array_equal(sc, ref["scales"].reshape(rows, -1)), e


@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
@pytest.mark.parametrize("shape", [(384, 2688), (256, 4096), (100, 48), (130, 1856)])
def test_quantize_grouped_equals_per_expert_oracle(mode, shape):
    E = 4
    x = bf16_stack(E, shape, sum(shape), [1.0, 0.02, 3.5, 1e-3])
    cfg = f46.QuantConfig(scale_mode=mode)
    gq = f46.quantize_grouped(x.cuda(), cfg)
    assert gq.codes.shape == (E, shape[0], -(-shape[1] // 16) * 8)
    for e in range(E):
        check_group(gq, e, O.quantize(bits(x[e]), mode), *shape)


def test_quantize_grouped_fp32_and_tie_directions():
    # experts whose amax gives alpha exact / rounded up / rounded down
    E, shape = 3, (256, 4096)
    x = bf16_stack(E, shape, 9, [0.5, 0.5, 0.5])
    for e, a in enumerate((5.25, 5.3125, 5.75)):
        x[e, 3, 7] = a
    gq = f46.quantize_grouped(x.cuda(), f46.QuantConfig(scale_mode="adaptive"))
    for e in range(E):
        check_group(gq, e, O.quantize(bits(x[e]), "adaptive"), *shape)
    xf = x.float() * 1.37
    gq = f46.quantize_grouped(xf.cuda(), f46.QuantConfig(scale_mode="adaptive"))
    for e in range(E):
        check_group(gq, e, O.quantize(xf[e].numpy(), "adaptive"), *shape)


def test_quantize_grouped_rejects_nonfinite():
    x = bf16_stack(2, (64, 64), 1, [1.0, 1.0])
    x[1, 5, 5] = float("inf")
    with pytest.raises(f46.InvalidInputError):
        f46.quantize_grouped(x.cuda(), f46.QuantConfig(scale_mode="adaptive"))


@pytest.mark.parametrize("shape", [(192, 320), (1856, 2688), (40, 72)])
def test_weights_2d_grouped_equals_per_expert(shape):
    E = 3 if shape[0] < 1000 else 2
    w = bf16_stack(E, shape, 3, [0.02, 0.05, 1.0])
    cfg = f46.QuantConfig(scale_mode="adaptive")
    gq = f46.quantize_weights_2d_grouped(w.cuda(), cfg)
    for e in range(E):
        one = f46.quantize_weights_2d(w[e].cuda(), cfg)
        q = gq.group(e)
        assert float(q.alpha_dev.item()) == one.alpha
        assert torch.equal(q.packed_codes, one.packed_codes)
        assert torch.equal(q.scales_tc, one.scales_tc)
        qt = gq.transposed.group(e)
        assert torch.equal(qt.packed_codes, one.transposed.packed_codes)
        assert torch.equal(qt.scales_tc, one.transposed.scales_tc)
    if shape[0] < 1000:  # the tile codes against the oracle directly
        ref = O.quantize_2d(bits(w[0]), "adaptive")
        assert np.array_equal(gq.group(0).packed_codes.cpu().numpy(), ref["codes"])


def wgrad_ref(a_bf16: torch.Tensor, spec, mode):
    """oracle: apply_rht(a.T) in float64 then the float64 quantizer."""
    a64 = a_bf16.float().double().numpy()
    y = O.apply_rht(np.ascontiguousarray(a64.T), spec.signs)
    return O.quantize(y, mode)


@pytest.mark.parametrize("mode", ["adaptive", "fixed6"])
@pytest.mark.parametrize("T,H", [(256, 320), (3072, 192), (64, 70), (48, 2688), (96, 200), (32, 8)])
def test_wgrad_operand_grouped_oracle(mode, T, H):
    E = 3
    a = bf16_stack(E, (T, H), T + H, [1.0, 1e-3, 2.5])
    cfg = f46.QuantConfig(scale_mode=mode, seed=4)
    spec = f46.RhtSpec(seed=cfg.seed)
    gq = f46.quantize_wgrad_operand_grouped(a.cuda(), cfg, spec)
    assert gq.shape == (H, T)
    for e in range(E):
        check_group(gq, e, wgrad_ref(a[e], spec, mode), H, T)


def test_wgrad_operand_exact_fallback_and_signed_zeros():
    # groups whose RHT values are not float32-exact (tiny next to large), all-zero
    # columns (signed zeros through the sign flips) and negative zeros
    T, H = 64, 64
    a = bf16_stack(1, (T, H), 17, [1.0])
    a[0, :16, 3] = 0.0
    a[0, :16, 4] = -0.0
    a[0, 16, 5] = 1e-30
    a[0, 17, 5] = 4.0
    a[0, 32:48, 6] = torch.tensor([1e-20] * 8 + [3.0] * 8, dtype=torch.bfloat16)
    cfg = f46.QuantConfig(scale_mode="adaptive", seed=1)
    spec = f46.RhtSpec(seed=1)
    gq = f46.quantize_wgrad_operand_grouped(a.cuda(), cfg, spec)
    check_group(gq, 0, wgrad_ref(a[0], spec, "adaptive"), H, T)


def test_wgrad_operand_matches_linear_wgrad_path():
    # the fused pass == the package's unfused apply_rht (float64) + quantize
    T, H = 128, 96
    a = bf16_stack(2, (T, H), 23, [1.0, 0.3])
    cfg = f46.QuantConfig(scale_mode="adaptive", seed=2)
    spec = f46.RhtSpec(seed=2)
    gq = f46.quantize_wgrad_operand_grouped(a.cuda(), cfg, spec)
    for e in range(2):
        y = f46.apply_rht(a[e].cuda().T.contiguous(), spec)
        q = f46.quantize_tensor_adaptive(y, cfg)
        assert torch.equal(gq.group(e).packed_codes, q.packed_codes)
        assert torch.equal(gq.group(e).scales_tc, q.scales_tc)
        assert float(gq.group(e).alpha_dev.item()) == q.alpha


def test_quantize_grouped_scale_ties_mixed_directions():
    """Experts whose tensor scales round up, down and exactly, each with block
    maxima on exact E4M3 ties of its own unrounded scale, in one grouped launch."""
    from tests.test_gpu_quant import scale_tie_tensor
    amaxes = (7.0, 6.5, 5.25, 0.109375)
    x = torch.stack([scale_tie_tensor(a, 5 + i) for i, a in enumerate(amaxes)])
    gq = f46.quantize_grouped(x.cuda(), f46.QuantConfig(scale_mode="adaptive"))
    for e in range(len(amaxes)):
        check_group(gq, e, O.quantize(bits(x[e]), "adaptive"), 512, 4096)
