"""GPU parity of the 4/6 quantize / dequantize path against the oracle.

Every comparison is bit-exact: FP4 codes (packed), E4M3 scales, the per-block
4-vs-6 choice and alpha; dequantized float64 values are exact and float32
values are the exact value rounded once (np.float32 of the reference).
Calls go through the package API -> C ABI (libfouroversix.so).
"""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from oracle import oracle as O
from tests.golden_util import opt, quant_cases

pytestmark = pytest.mark.gpu

CASES = quant_cases()


def to_torch(x: np.ndarray) -> torch.Tensor:
    if x.dtype == np.uint16:
        return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run(x_t, mode, rule="mse", alpha=None, fp8_cap=None):
    kw = dict(want_rowmajor=True, want_pick4=True)
    if mode == "adaptive":
        return f46.quantize_tensor_adaptive(x_t, f46.QuantConfig(scale_mode="adaptive", rule=rule),
                                            alpha=alpha, **kw)
    cfg = f46.QuantConfig(scale_mode=mode, **({} if fp8_cap is None else {"fp8_cap": fp8_cap}))
    return f46.quantize_tensor(x_t, cfg, alpha=alpha, **kw)


def assert_same(q, ref, rows):
    assert q.alpha == ref["alpha"]
    assert np.array_equal(q.scales_rm.cpu().numpy(), ref["scales"].reshape(rows, -1))
    got = q.packed_codes.cpu().numpy()
    bad = np.argwhere(got != ref["codes"])
    assert bad.size == 0, f"{len(bad)} code bytes differ, first at {bad[:4].tolist()}"
    assert np.array_equal(q.pick4.cpu().numpy(), ref["pick4"].reshape(rows, -1))


@pytest.mark.parametrize("name,rec", CASES, ids=[c[0] for c in CASES])
def test_golden_fixture(name, rec):
    x = rec["x"]
    cols = x.shape[-1]
    rows = x.size // cols
    q = run(to_torch(x), str(rec["mode"]), str(rec["rule"]), opt(rec["alpha_override"]),
            opt(rec["fp8_cap"]))
    assert q.shape == tuple(x.shape)
    assert_same(q, rec, rows)
    # tcgen05-layout scales agree with the row-major view
    assert np.array_equal(f46.blockquant.tc_to_rowmajor(q.scales_tc, rows, q.nblocks_per_row).cpu().numpy(),
                          rec["scales"].reshape(rows, -1))
    if "deq" in rec:
        d64 = f46.dequantize_tensor(q, torch.float64).cpu().numpy().reshape(-1)
        assert np.array_equal(d64, rec["deq"])
        d32 = f46.dequantize_tensor(q, torch.float32).cpu().numpy().reshape(-1)
        assert np.array_equal(d32, rec["deq"].astype(np.float32))


def bf16_randn(shape, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(*shape, generator=g) * std).to(torch.bfloat16)


def bits(x: torch.Tensor) -> np.ndarray:
    return x.view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c1_4096sq_bf16_bit_exact(mode, seed):
    """Config 1: 4096x4096 Gaussian BF16 (seed 2 has amax 5.75 -> alpha inexact)."""
    x = bf16_randn((4096, 4096), seed)
    q = run(x.cuda(), mode)
    ref = O.quantize(bits(x), mode)
    assert_same(q, ref, 4096)


@pytest.mark.parametrize("shape", [(4096, 14336), (14336, 4096)])
def test_c2_llama_weight_shapes(shape):
    """Config 2: Llama-3-8B linear weights, N(0, 0.02^2) BF16."""
    x = bf16_randn(shape, 7, std=0.02)
    q = run(x.cuda(), "adaptive")
    ref = O.quantize(bits(x), "adaptive")
    assert_same(q, ref, shape[0])


def test_fp32_input_bit_exact():
    g = torch.Generator().manual_seed(5)
    x = torch.randn(1024, 1536, generator=g) * 3
    q = run(x.cuda(), "adaptive")
    ref = O.quantize(x.numpy(), "adaptive")
    assert_same(q, ref, 1024)


@pytest.mark.parametrize("shape", [(5,), (3, 7), (2, 3, 40), (17, 33), (300, 80), (129, 4160)])
def test_ragged_shapes(shape):
    x = bf16_randn(shape, 3)
    q = run(x.cuda(), "adaptive")
    x2 = bits(x).reshape(-1, shape[-1])
    ref = O.quantize(x2, "adaptive")
    assert_same(q, ref, x2.shape[0])


def test_nonfinite_rejected():
    x = torch.randn(64, 64).to(torch.bfloat16)
    x[3, 5] = float("inf")
    with pytest.raises(f46.InvalidInputError):
        run(x.cuda(), "adaptive")
    x[3, 5] = float("nan")
    with pytest.raises(f46.InvalidInputError):
        run(x.cuda(), "adaptive", alpha=1.0)


def test_idempotent_requantization():
    # test_blockquant.py:182-189, on the GPU
    x = (bf16_randn((256, 512), 13) * 2.5).float()
    q1 = f46.quantize_tensor(x.cuda(), f46.QuantConfig())
    q2 = f46.quantize_tensor(f46.dequantize_tensor(q1, torch.float64), f46.QuantConfig())
    assert q1 == q2


def test_alpha_override_validation():
    x = torch.ones(1, 16).cuda()
    with pytest.raises(f46.InvalidInputError):
        f46.quantize_tensor(x, f46.QuantConfig(), alpha=-1.0)
    with pytest.raises(f46.InvalidInputError):
        f46.quantize_tensor(x, f46.QuantConfig(), alpha=float("inf"))


def f64_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round float64 to bf16 once (RNE): round-to-odd to float32, then RNE."""
    f = np.asarray(f, np.float64)
    rn = f.astype(np.float32)
    away = np.abs(rn.astype(np.float64)) > np.abs(f)
    rz = np.where(away, np.nextafter(rn, np.float32(0)), rn)
    b = rz.view(np.uint32).copy()
    b |= (rz.astype(np.float64) != f).astype(np.uint32)
    return ((b.astype(np.uint64) + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def test_dequant_bf16_is_single_rounding():
    x = bf16_randn((512, 1024), 21)
    q = run(x.cuda(), "adaptive")
    d64 = f46.dequantize_tensor(q, torch.float64).cpu().numpy()
    d16 = f46.dequantize_tensor(q, torch.bfloat16).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(d16, f64_to_bf16_bits(d64))


def test_nan_scale_rejected_on_dequant():
    q = f46.QuantizedTensor(shape=(16,), fmt="nvfp4", alpha=1.0,
                            scale_codes=np.array([[0x7F]], dtype=np.uint8),
                            codes=np.zeros(16, dtype=np.uint8))
    with pytest.raises(f46.InvalidInputError):
        f46.dequantize_tensor(q)


def test_reference_style_float64_inputs():
    # the reference's own tests feed float64 Gaussians; the exact path takes them
    rng = np.random.Generator(np.random.Philox(3))
    X = rng.standard_normal((8, 48))
    q = f46.quantize_tensor(X, f46.QuantConfig())
    ref = O.quantize(X, "fixed6")
    assert q.alpha == ref["alpha"]
    assert np.array_equal(q.packed_codes.cpu().numpy(), ref["codes"])
    D = f46.dequantize_tensor(q, torch.float64).cpu().numpy()
    assert np.array_equal(D, O.dequantize(ref["codes"], ref["scales"], ref["alpha"], 8, 48))


# 0.008766868151724339 is a float32 for which RN32(11 * alpha) is an inexact bf16
# midpoint: bf16 output must take the round-to-odd route (DQ_ODD)
@pytest.mark.parametrize("alpha", [None, 0.003, 0.008766868151724339])
@pytest.mark.parametrize("shape", [(5, 48), (1, 16), (3, 1040), (33, 4112), (64, 1024), (257, 2064),
                                   (130, 272)])
@pytest.mark.parametrize("path", ["tma", "vec"])
def test_dequant_flat_paths_ragged(shape, alpha, path, test_hook):
    """K3's TMA-staged and coalesced variants on chunk- and row-ragged shapes
    (odd blocks per row too), with f32-exact alphas (direct and round-to-odd
    bf16 routes) and an f64-only alpha: f32 is the exact value rounded once,
    bf16 likewise (a single rounding of the float64 value)."""
    if path == "vec":
        test_hook("dq_vec", 1)
    x = bf16_randn(shape, shape[0] * 31 + shape[1])
    q = run(x.cuda(), "adaptive", alpha=alpha)
    d64 = f46.dequantize_tensor(q, torch.float64).cpu().numpy()
    d32 = f46.dequantize_tensor(q, torch.float32).cpu().numpy()
    assert np.array_equal(d32, d64.astype(np.float32))
    d16 = f46.dequantize_tensor(q, torch.bfloat16).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(d16, f64_to_bf16_bits(d64))


@pytest.mark.parametrize("mode", ["adaptive", "fixed6"])
def test_k2_multi_launch_row_slabs(mode, test_hook):
    """K2 keeps 32-bit offsets and launches at most 2^31 input bytes at a time
    in 128-row slabs; forcing 1 MB slabs (4 launches + a ragged last slab)
    gives the single-launch container bit for bit."""
    x = bf16_randn((1000, 512), 5).cuda()
    ref = run(x, mode)
    test_hook("seg_chunk_bytes", 1 << 18)
    got = run(x, mode)
    assert got.alpha == ref.alpha
    assert torch.equal(got.packed_codes, ref.packed_codes)
    assert torch.equal(got.scales_tc, ref.scales_tc)
    assert torch.equal(got.pick4, ref.pick4) and torch.equal(got.scales_rm, ref.scales_rm)


def tie_direction(amax: float, mcap: float) -> int:
    """Sign of RN32(amax/mcap)*mcap - amax (f46_device.cuh tie_direction):
    -1 when alpha rounds up, +1 when it rounds down, 0 when it is exact."""
    a = float(np.float32(np.float32(amax) / np.float32(mcap)))
    d = a * mcap - amax
    return -1 if d > 0 else (1 if d < 0 else 0)


# amax values whose alpha = RN32(amax / 1536) is exact (0), rounded up (-1) or
# rounded down (+1); the streaming kernel is specialised on that direction.
TIE_AMAX = [6.0, 7.5, 5.25, 5.75, 5.3125, 6.5, 7.0, 5.1875]


@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
@pytest.mark.parametrize("amax", TIE_AMAX)
def test_timed_instantiation_every_tie_direction(mode, amax):
    """The instantiation bench.py times (no row-major scales, no pick4 output,
    whole 2048-element segments) against the oracle, bit for bit, for tensors
    of every tensor-wide tie direction (TDIR -1, 0, +1): packed codes and
    tcgen05-layout scales."""
    x = bf16_randn((512, 4096), int(amax * 64), std=0.5)
    x[7, 100] = amax
    x[300, 5] = -amax
    q = f46.quantize_tensor_adaptive(x.cuda(), f46.QuantConfig(scale_mode="adaptive")) \
        if mode == "adaptive" else f46.quantize_tensor(x.cuda(), f46.QuantConfig(scale_mode=mode))
    ref = O.quantize(bits(x), mode)
    assert q.alpha == ref["alpha"]
    got = q.packed_codes.cpu().numpy()
    bad = np.argwhere(got != ref["codes"])
    assert bad.size == 0, f"{len(bad)} code bytes differ, first at {bad[:4].tolist()}"
    sc = f46.blockquant.tc_to_rowmajor(q.scales_tc, 512, 256).cpu().numpy()
    assert np.array_equal(sc, ref["scales"].reshape(512, -1))


def test_tie_amax_cover_every_direction():
    assert {tie_direction(a, 1536.0) for a in TIE_AMAX} == {-1, 0, 1}


@pytest.mark.parametrize("mode", ["adaptive", "fixed6"])
@pytest.mark.parametrize("shape", [(300, 2688), (129, 48), (5, 16), (1000, 4160), (3, 1856), (257, 272)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_timed_instantiation_flat_tiles(mode, shape, dtype):
    """Row lengths that are not a multiple of the 2048-element tile take the
    flat streaming loop (tiles of 128 consecutive blocks across rows, a short
    last tile): codes and tcgen05 scales against the oracle."""
    g = torch.Generator().manual_seed(shape[0] + shape[1])
    x = (torch.randn(*shape, generator=g) * 1.7).to(dtype)
    cfg = f46.QuantConfig(scale_mode=mode)
    q = (f46.quantize_tensor_adaptive(x.cuda(), cfg) if mode == "adaptive"
         else f46.quantize_tensor(x.cuda(), cfg))
    ref = O.quantize(bits(x) if dtype == torch.bfloat16 else x.numpy(), mode)
    assert q.alpha == ref["alpha"]
    assert np.array_equal(q.packed_codes.cpu().numpy(), ref["codes"])
    nb = -(-shape[1] // 16)
    sc = f46.blockquant.tc_to_rowmajor(q.scales_tc, shape[0], nb).cpu().numpy()
    assert np.array_equal(sc, ref["scales"].reshape(shape[0], -1))


@pytest.mark.parametrize("shape", [(4096, 4096), (300, 2688), (17, 48), (1024, 14336)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("mode", ["adaptive", "fixed4"])
def test_fused_single_launch_equals_two_kernels(shape, dtype, mode):
    """f46_quantize_fused (amax and quantize in one cooperative launch, the
    path quantize_tensor* takes for L2-sized tensors) == f46_amax +
    f46_quantize, and both == the oracle."""
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import scales_tc_bytes
    g = torch.Generator().manual_seed(shape[1])
    x = (torch.randn(*shape, generator=g) * 0.7).to(dtype).cuda()
    L = _lib.load()
    rows, cols = shape
    mcap = {"adaptive": 1536.0, "fixed4": 1792.0}[mode]
    dt = _lib.DT_BF16 if dtype == torch.bfloat16 else _lib.DT_F32
    outs = []
    for fused in (True, False):
        codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device="cuda")
        sc = torch.zeros(scales_tc_bytes(rows, cols), dtype=torch.uint8, device="cuda")
        alpha = torch.empty(1, dtype=torch.float64, device="cuda")
        work = torch.zeros(2, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        if fused:
            assert L.f46_quantize_fused(x.data_ptr(), dt, rows, cols, _lib.MODE[mode], 0, mcap,
                                        work.data_ptr(), codes.data_ptr(), sc.data_ptr(),
                                        alpha.data_ptr(), None, s) == 0
        else:
            assert L.f46_amax(x.data_ptr(), dt, x.numel(), work.data_ptr(), s) == 0
            assert L.f46_quantize(x.data_ptr(), dt, rows, cols, _lib.MODE[mode], 0, mcap,
                                  work.data_ptr(), 0.0, codes.data_ptr(), sc.data_ptr(), None, None,
                                  alpha.data_ptr(), None, s) == 0
        outs.append((codes, sc, alpha, work[0].clone()))
    (c1, s1, a1, m1), (c2, s2, a2, m2) = outs
    assert torch.equal(m1, m2) and torch.equal(a1, a2)
    assert torch.equal(c1, c2) and torch.equal(s1, s2)
    ref = O.quantize(bits(x.cpu()) if dtype == torch.bfloat16 else x.cpu().numpy(), mode)
    assert float(a1.item()) == ref["alpha"]
    assert np.array_equal(c1.cpu().numpy(), ref["codes"])


def scale_tie_tensor(amax: float, seed: int) -> torch.Tensor:
    """512x4096 BF16 whose block maxima sit on exact E4M3 ties of the
    unrounded scale amax/mcap for every mode: significands 7*(17..31) and
    49, 63 (adaptive, amax = 7*2^e) and 17..31 (fixed6), at several binades."""
    g = torch.Generator().manual_seed(seed)
    x = torch.rand(512, 4096, generator=g) * 2.0 - 1.0
    sig = torch.tensor([7 * t for t in range(17, 32, 2)] + [49, 63] + list(range(17, 32, 2)),
                       dtype=torch.float32)
    nb = 512 * 256
    pick = sig[torch.randint(0, len(sig), (nb,), generator=g)]
    expo = torch.randint(-14, -7, (nb,), generator=g).float()
    sgn = torch.where(torch.rand(nb, generator=g) < 0.5, -1.0, 1.0)
    bmax = sgn * pick * torch.exp2(expo) * (amax / 7.0)
    xb = x.view(nb, 16) * bmax.abs().unsqueeze(1) * 0.9
    xb[:, 0] = bmax
    x = xb.view(512, 4096).to(torch.bfloat16)
    x[7, 100] = amax
    return x


@pytest.mark.parametrize("mode", ["adaptive", "fixed6", "fixed4"])
@pytest.mark.parametrize("amax", [7.0, 3.5, 0.109375, 5.25, 6.5])
def test_scale_code_ties_follow_tie_direction(mode, amax):
    """Block scales on exact E4M3 ties of the unrounded tensor scale: the
    streaming kernel settles them by the tensor-wide tie direction (no
    deferral); codes and scales equal the oracle's bit for bit."""
    x = scale_tie_tensor(amax, int(amax * 1000))
    cfg = f46.QuantConfig(scale_mode=mode)
    q = f46.quantize_tensor_adaptive(x.cuda(), cfg) if mode == "adaptive" else \
        f46.quantize_tensor(x.cuda(), cfg)
    ref = O.quantize(bits(x), mode)
    assert q.alpha == ref["alpha"]
    got = q.packed_codes.cpu().numpy()
    bad = np.argwhere(got != ref["codes"])
    assert bad.size == 0, f"{len(bad)} code bytes differ, first at {bad[:4].tolist()}"
    sc = f46.blockquant.tc_to_rowmajor(q.scales_tc, 512, 256).cpu().numpy()
    assert np.array_equal(sc, ref["scales"].reshape(512, -1))


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_parallel_resolver_special_blocks(fused, dtype):
    """Small tensors resolve their deferred blocks 16 lanes per block (odd and
    even list lengths, special blocks: all-zero with signed zeros, values
    below the fast path's range, near-ties of every kind); fused and
    two-kernel launches both equal the oracle bit for bit."""
    from paper_2512_02010_b200 import _lib
    from paper_2512_02010_b200.blockquant import scales_tc_bytes, tc_to_rowmajor
    rows, cols = 384, 2048
    g = torch.Generator().manual_seed(77)
    x = torch.randn(rows, cols, generator=g)
    nb = rows * cols // 16
    xb = x.view(nb, 16)
    kind = torch.randint(0, 6, (nb,), generator=g)
    xb[kind == 0] = 0.0
    xb[kind == 1] = -0.0
    xb[kind == 2] *= 1e-13          # bmax below 2^-40: exact path
    xb[kind == 3] = torch.round(xb[kind == 3] * 4) / 4  # many values on the FP4 grid / ties
    x[5, 7] = 6.0
    x = x.to(dtype)
    ref = O.quantize(bits(x) if dtype == torch.bfloat16 else x.numpy(), "adaptive")
    L = _lib.load()
    dt = _lib.DT_BF16 if dtype == torch.bfloat16 else _lib.DT_F32
    xc = x.cuda()
    codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device="cuda")
    sc = torch.zeros(scales_tc_bytes(rows, cols), dtype=torch.uint8, device="cuda")
    alpha = torch.empty(1, dtype=torch.float64, device="cuda")
    work = torch.zeros(2, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    if fused:
        assert L.f46_quantize_fused(xc.data_ptr(), dt, rows, cols, _lib.MODE["adaptive"], 0, 1536.0,
                                    work.data_ptr(), codes.data_ptr(), sc.data_ptr(),
                                    alpha.data_ptr(), None, s) == 0
    else:
        assert L.f46_amax(xc.data_ptr(), dt, xc.numel(), work.data_ptr(), s) == 0
        assert L.f46_quantize(xc.data_ptr(), dt, rows, cols, _lib.MODE["adaptive"], 0, 1536.0,
                              work.data_ptr(), 0.0, codes.data_ptr(), sc.data_ptr(), None, None,
                              alpha.data_ptr(), None, s) == 0
    torch.cuda.synchronize()
    assert float(alpha.item()) == ref["alpha"]
    got = codes.cpu().numpy()
    bad = np.argwhere(got != ref["codes"])
    assert bad.size == 0, f"{len(bad)} code bytes differ, first at {bad[:4].tolist()}"
    rm = tc_to_rowmajor(sc, rows, cols // 16).cpu().numpy()
    assert np.array_equal(rm, ref["scales"].reshape(rows, -1))
