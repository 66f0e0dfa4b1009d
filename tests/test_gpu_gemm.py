"""GPU parity of the tcgen05 NVFP4 GEMM (f46_gemm_nvfp4) -- the consumer of
the quantized containers, reference qlinear.py:74-93 emulated_fp4_matmul.

Oracle: the exact float64 product of the exactly dequantized operands (the
CPU oracle's dequantization for small shapes, the GPU's own float64
dequantization -- bit-identical to the oracle, see test_gpu_quant -- for large
ones).  Tolerance: relative Frobenius error <= 1e-5, the reference's own bound
(test_acceptance.py:191-198); identity operands must be exact.
"""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from oracle import oracle as O
from tests.golden_util import load

pytestmark = pytest.mark.gpu

ADAPT = f46.QuantConfig(scale_mode="adaptive")
REL_TOL = 1e-5


def bf16_randn(shape, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(*shape, generator=g) * std).to(torch.bfloat16)


def rel_fro(got, ref):
    got = got.double()
    ref = ref.double()
    return float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))


GEMMS = load("golden_gemm.npz")


@pytest.mark.parametrize("name,rec", GEMMS, ids=[c[0] for c in GEMMS])
def test_golden_reference_matmul(name, rec):
    """Reference emulated_fp4_matmul outputs (tests/golden/make_golden.py)."""
    a = torch.from_numpy(rec["a"].view(np.int16).copy()).view(torch.bfloat16).cuda()
    b = torch.from_numpy(rec["b"].view(np.int16).copy()).view(torch.bfloat16).cuda()
    aq = f46.quantize_tensor_adaptive(a, ADAPT)
    bq = f46.quantize_tensor_adaptive(b, ADAPT)
    got = f46.emulated_fp4_matmul(aq, bq, transpose_b=True)
    ref = torch.from_numpy(rec["c"]).cuda()
    assert got.dtype == torch.float32 and got.shape == ref.shape
    assert rel_fro(got, ref) <= REL_TOL


def oracle_product(x: torch.Tensor, w: torch.Tensor):
    """float64 dequant(q(x)) @ dequant(q(w))^T from the CPU oracle."""
    bx = x.view(torch.int16).numpy().view(np.uint16)
    bw = w.view(torch.int16).numpy().view(np.uint16)
    rx, rw = O.quantize(bx, "adaptive"), O.quantize(bw, "adaptive")
    dx = O.dequantize(rx["codes"], rx["scales"], rx["alpha"], *x.shape)
    dw = O.dequantize(rw["codes"], rw["scales"], rw["alpha"], *w.shape)
    return torch.from_numpy(dx @ dw.T)


@pytest.mark.parametrize("M,N,K", [(128, 256, 256), (256, 512, 1024), (200, 300, 320), (64, 80, 48), (33, 70, 208),
                                   (1, 16, 64), (130, 260, 96), (384, 256, 4096)])
def test_matches_oracle_small(M, N, K):
    x = bf16_randn((M, K), M + K)
    w = bf16_randn((N, K), N + 7)
    got = f46.emulated_fp4_matmul(f46.quantize_tensor_adaptive(x.cuda(), ADAPT),
                                  f46.quantize_tensor_adaptive(w.cuda(), ADAPT), transpose_b=True)
    assert rel_fro(got.cpu(), oracle_product(x, w)) <= REL_TOL


def gpu_oracle(aq, bq):
    a = f46.dequantize_tensor(aq, torch.float64)
    b = f46.dequantize_tensor(bq, torch.float64)
    return a @ b.T


@pytest.mark.parametrize("M,N,K", [(3072, 1856, 2688), (3072, 2688, 1856), (2048, 2048, 8192)])
def test_moe_and_large_shapes(M, N, K):
    """Nemotron-3-Nano expert shapes (hidden 2688, FFN 1856: N not a multiple of
    256, K not a multiple of 256) and a deep-K case."""
    x = bf16_randn((M, K), 11).cuda()
    w = (bf16_randn((N, K), 12) * 0.02).to(torch.bfloat16).cuda()
    aq = f46.quantize_tensor_adaptive(x, ADAPT)
    bq = f46.quantize_tensor_adaptive(w, ADAPT)
    got = f46.emulated_fp4_matmul(aq, bq, transpose_b=True)
    assert rel_fro(got, gpu_oracle(aq, bq)) <= REL_TOL


def identity_container(n: int) -> f46.QuantizedTensor:
    """Exact n x n identity: diagonal code 0b0010 (1.0), unit scales
    (test_qlinear.py:23-31)."""
    codes = np.zeros((n, n), dtype=np.uint8)
    np.fill_diagonal(codes, 0b0010)
    return f46.QuantizedTensor(shape=(n, n), fmt="nvfp4", alpha=1.0,
                               scale_codes=np.full((n, n // 16), 0x38, dtype=np.uint8),
                               codes=codes)


@pytest.mark.parametrize("rows,n", [(16, 64), (200, 256), (128, 512)])
def test_identity_operand_is_exact(rows, n):
    """A @ I^T == dequant(A) exactly (test_qlinear.py:67-71, TN form): pins the
    code nibble order and the tcgen05 scale-factor layout."""
    aq = f46.quantize_tensor_adaptive(bf16_randn((rows, n), 61).cuda(), ADAPT)
    got = f46.emulated_fp4_matmul(aq, identity_container(n), transpose_b=True)
    assert torch.equal(got, f46.dequantize_tensor(aq, torch.float32))


def test_bf16_out_is_post_rounding():
    aq = f46.quantize_tensor_adaptive(bf16_randn((256, 512), 63).cuda(), ADAPT)
    bq = f46.quantize_tensor_adaptive(bf16_randn((384, 512), 64).cuda(), ADAPT)
    wide = f46.emulated_fp4_matmul(aq, bq, transpose_b=True)
    narrow = f46.emulated_fp4_matmul(aq, bq, transpose_b=True, bf16_out=True)
    assert torch.equal(narrow, f46.round_to_bf16(wide))


def test_non_tn_layout_matches_dequant_product():
    aq = f46.quantize_tensor(bf16_randn((64, 96), 65).cuda(), f46.QuantConfig())
    bq = f46.quantize_tensor(bf16_randn((96, 48), 66).cuda(), f46.QuantConfig())
    got = f46.emulated_fp4_matmul(aq, bq)
    ref = f46.dequantize_tensor(aq, torch.float64) @ f46.dequantize_tensor(bq, torch.float64)
    assert rel_fro(got, ref) <= REL_TOL


def test_inner_dim_mismatch_and_rank():
    aq = f46.quantize_tensor(bf16_randn((4, 32), 1).cuda(), f46.QuantConfig())
    bq = f46.quantize_tensor(bf16_randn((4, 16), 2).cuda(), f46.QuantConfig())
    with pytest.raises(f46.InvalidInputError):
        f46.emulated_fp4_matmul(aq, bq, transpose_b=True)
    vq = f46.quantize_tensor(torch.ones(16).cuda(), f46.QuantConfig())
    with pytest.raises(f46.InvalidInputError):
        f46.emulated_fp4_matmul(vq, bq)


def test_grouped_matches_per_group():
    G, M, N, K = 3, 384, 320, 512
    qa = [f46.quantize_tensor_adaptive(bf16_randn((M, K), 100 + i).cuda(), ADAPT) for i in range(G)]
    qb = [f46.quantize_tensor_adaptive(bf16_randn((N, K), 200 + i).cuda(), ADAPT) for i in range(G)]
    st = lambda xs: torch.stack(xs)
    out = f46.gemm_nvfp4_grouped(st([q.packed_codes for q in qa]), st([q.scales_tc for q in qa]),
                                 torch.cat([q.alpha_dev for q in qa]),
                                 st([q.packed_codes for q in qb]), st([q.scales_tc for q in qb]),
                                 torch.cat([q.alpha_dev for q in qb]), M, N, K)
    for i in range(G):
        assert torch.equal(out[i], f46.gemm_nvfp4(qa[i], qb[i]))


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_persistent_and_simple_kernels_agree(out_dtype, test_hook):
    """The CTA-pair kernel (default), the single-CTA persistent kernel
    (test hook gemm_kernel 1) and the one-tile-per-CTA kernel (gemm_kernel 2) accumulate
    every output element over K in the same order: identical bits, also into
    a strided output (ldc = N + 1)."""
    M, N, K = 700, 1000, 1024
    aq = f46.quantize_tensor_adaptive(bf16_randn((M, K), 71).cuda(), ADAPT)
    bq = f46.quantize_tensor_adaptive(bf16_randn((N, K), 72).cuda(), ADAPT)
    fast = f46.gemm_nvfp4(aq, bq, out_dtype)
    wide = torch.empty((M, N + 1), dtype=out_dtype, device="cuda")
    strided = f46.gemm_nvfp4(aq, bq, out_dtype, out=wide[:, :N])
    test_hook("gemm_kernel", 1)
    one_sm = f46.gemm_nvfp4(aq, bq, out_dtype)
    test_hook("gemm_kernel", 2)
    simple = f46.gemm_nvfp4(aq, bq, out_dtype)
    assert torch.equal(one_sm, simple)
    assert torch.equal(fast, strided)
    assert torch.equal(fast, simple), "CTA-pair and single-CTA kernels differ"
    assert rel_fro(fast.float(), gpu_oracle(aq, bq)) <= (REL_TOL if out_dtype == torch.float32 else 4e-3)


@pytest.mark.parametrize("kernel", ["pair", "1sm", "simple"])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("M,N,K", [(700, 1000, 1024), (256, 512, 256), (33, 40, 48)])
def test_producer_fused_amax(M, N, K, out_dtype, kernel, test_hook):
    """The epilogue's amax equals max |C| of the stored tensor exactly (every
    kernel, every output type, ragged tiles) and, handed to the next quantize
    as its amax, yields the container K1 + K2 produce."""
    test_hook("gemm_kernel", {"pair": 0, "1sm": 1, "simple": 2}[kernel])
    aq = f46.quantize_tensor_adaptive(bf16_randn((M, K), 81).cuda(), ADAPT)
    bq = f46.quantize_tensor_adaptive(bf16_randn((N, K), 82).cuda(), ADAPT)
    amax = torch.full((1,), 123.0, dtype=torch.float64, device="cuda")  # zeroed by the call
    c = f46.gemm_nvfp4(aq, bq, out_dtype, amax_out=amax)
    assert torch.equal(c, f46.gemm_nvfp4(aq, bq, out_dtype))
    assert float(amax) == float(c.abs().max().double())
    if out_dtype == torch.bfloat16 and c.shape[1] % 16 == 0:
        fused = f46.quantize_tensor_adaptive(c, ADAPT, d_amax=amax)
        plain = f46.quantize_tensor_adaptive(c, ADAPT)
        assert fused.alpha == plain.alpha
        assert torch.equal(fused.packed_codes, plain.packed_codes)
        assert torch.equal(fused.scales_tc, plain.scales_tc)


def test_grouped_amax_per_group():
    G, M, N, K = 3, 300, 256, 256
    qa = [f46.quantize_tensor_adaptive(bf16_randn((M, K), 300 + i, std=1.0 + i).cuda(), ADAPT)
          for i in range(G)]
    qb = [f46.quantize_tensor_adaptive(bf16_randn((N, K), 400 + i).cuda(), ADAPT) for i in range(G)]
    st = lambda xs: torch.stack(xs)
    amax = torch.empty(G, dtype=torch.float64, device="cuda")
    out = f46.gemm_nvfp4_grouped(st([q.packed_codes for q in qa]), st([q.scales_tc for q in qa]),
                                 torch.cat([q.alpha_dev for q in qa]),
                                 st([q.packed_codes for q in qb]), st([q.scales_tc for q in qb]),
                                 torch.cat([q.alpha_dev for q in qb]), M, N, K, torch.bfloat16,
                                 amax_out=amax)
    for g in range(G):
        assert float(amax[g]) == float(out[g].abs().max().double())
    with pytest.raises(f46.InvalidInputError):
        f46.gemm_nvfp4(qa[0], qb[0], amax_out=torch.zeros(2, dtype=torch.float64, device="cuda"))
