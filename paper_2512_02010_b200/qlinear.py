"""NVFP4 GEMM consumer of the quantized containers.

Mirrors the reference's fp4emu.qlinear (/root/reference/pkg/src/fp4emu/
qlinear.py): ``emulated_fp4_matmul`` (:74-93) and ``round_to_bf16`` (:56-61).

``emulated_fp4_matmul(aq, bq, transpose_b=True)`` -- both operands blocked
along K, the layout of every NVFP4 linear layer (FPROP x @ W^T, WGRAD) -- runs
on the B200's tensor cores: ``f46_gemm_nvfp4`` issues tcgen05.mma
kind::mxf4nvf4 directly on the packed E2M1 codes and the tcgen05-layout E4M3
scales the quantizer wrote, with alpha_a * alpha_b applied in the epilogue.
The reference dequantizes to float32 and accumulates in float32 in ascending
k; the tensor cores accumulate the same exact products in float32 in their own
order, so results agree to float32 accumulation error (relative Frobenius
<= 1e-5, the reference's own bound, test_acceptance.py:191-198).

``transpose_b=False`` asks for dequant(A) @ dequant(B) with B blocked along N,
which no block-scaled tensor-core instruction can consume; that case
dequantizes both operands on the GPU (f46_dequantize, rounded once to
float32 as the reference's ``astype(np.float32)``) and runs the reference's
ordered float32 accumulation (f46_matmul_f32_ordered) -- bit-identical to
``_accum_matmul_f32``.
"""

from __future__ import annotations

import torch

from . import _lib
from .blockquant import QuantizedTensor, _stream, dequantize_tensor
from .errors import ConfigError, InvalidInputError

__all__ = ["emulated_fp4_matmul", "gemm_nvfp4", "gemm_nvfp4_grouped", "linear_dgrad",
           "linear_forward", "linear_wgrad", "round_to_bf16"]


def round_to_bf16(x: torch.Tensor) -> torch.Tensor:
    """float32 -> bf16 -> float32, round to nearest even (qlinear.py:56-61)."""
    return x.to(torch.float32).to(torch.bfloat16).to(torch.float32)


def gemm_nvfp4(aq: QuantizedTensor, bq: QuantizedTensor, out_dtype=torch.float32,
               out: torch.Tensor | None = None,
               amax_out: torch.Tensor | None = None) -> torch.Tensor:
    """C[M,N] = dequant(aq) @ dequant(bq)^T on tcgen05 (both blocked along K).

    ``amax_out`` (a float64 CUDA tensor of one element): the epilogue also
    writes max |C| of the stored values into it (producer-fused amax), ready to
    pass as ``d_amax=`` to the next quantize so it skips its amax pass."""
    L = _lib.load()
    if len(aq.shape) != 2 or len(bq.shape) != 2:
        raise InvalidInputError("the NVFP4 GEMM is defined for 2-D operands")
    M, K = aq.shape
    N, Kb = bq.shape
    if K != Kb:
        raise InvalidInputError(f"inner dimensions differ: {aq.shape} x {tuple(bq.shape)}^T")
    dev = aq.scales_tc.device
    dt = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16}[out_dtype]
    if out is None:
        out = torch.empty((M, N), dtype=out_dtype, device=dev)
    a_codes, b_codes, k_eff = aq.packed_codes, bq.packed_codes, K
    if (-(-K // 16)) % 2:
        # TMA needs 16-byte code rows: append one all-zero 16-element block
        # (its scales are already zero in the tcgen05 layout's padding)
        a_codes = torch.nn.functional.pad(a_codes, (0, 8))
        b_codes = torch.nn.functional.pad(b_codes, (0, 8))
        k_eff = (-(-K // 16) + 1) * 16
    if amax_out is None:
        rc = L.f46_gemm_nvfp4(a_codes.data_ptr(), aq.scales_tc.data_ptr(),
                              aq.alpha_dev.data_ptr(), b_codes.data_ptr(),
                              bq.scales_tc.data_ptr(), bq.alpha_dev.data_ptr(), M, N, k_eff,
                              out.data_ptr(), out.stride(0), dt, _stream())
    else:
        _check_amax_buffer(amax_out, 1, dev)
        amax_out.zero_()
        rc = L.f46_gemm_nvfp4_amax(a_codes.data_ptr(), aq.scales_tc.data_ptr(),
                                   aq.alpha_dev.data_ptr(), b_codes.data_ptr(),
                                   bq.scales_tc.data_ptr(), bq.alpha_dev.data_ptr(), M, N, k_eff,
                                   out.data_ptr(), out.stride(0), dt, amax_out.data_ptr(),
                                   _stream())
    _lib.check(rc, "f46_gemm_nvfp4")
    return out


def _check_amax_buffer(t: torch.Tensor, n: int, dev) -> None:
    if (not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or t.numel() != n
            or t.device != dev or not t.is_contiguous()):
        raise InvalidInputError(f"amax_out must be a contiguous float64 CUDA tensor of {n} "
                                "element(s) on the operands' device")


def gemm_nvfp4_grouped(a_codes, a_scales, a_alpha, b_codes, b_scales, b_alpha, M, N, K,
                       out_dtype=torch.float32, amax_out: torch.Tensor | None = None) -> torch.Tensor:
    """G independent GEMMs of one shape (MoE experts): operands packed back to
    back ([G, ...] device tensors), one alpha per group, C is [G, M, N].
    ``amax_out`` (float64 [G]): per-group max |C| from the epilogue."""
    L = _lib.load()
    G = a_codes.shape[0]
    dt = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16}[out_dtype]
    out = torch.empty((G, M, N), dtype=out_dtype, device=a_codes.device)
    if amax_out is None:
        rc = L.f46_gemm_nvfp4_grouped(G, a_codes.data_ptr(), a_scales.data_ptr(),
                                      a_alpha.data_ptr(), b_codes.data_ptr(), b_scales.data_ptr(),
                                      b_alpha.data_ptr(), M, N, K, out.data_ptr(), N, dt, _stream())
    else:
        _check_amax_buffer(amax_out, G, a_codes.device)
        amax_out.zero_()
        rc = L.f46_gemm_nvfp4_grouped_amax(G, a_codes.data_ptr(), a_scales.data_ptr(),
                                           a_alpha.data_ptr(), b_codes.data_ptr(),
                                           b_scales.data_ptr(), b_alpha.data_ptr(), M, N, K,
                                           out.data_ptr(), N, dt, amax_out.data_ptr(), _stream())
    _lib.check(rc, "f46_gemm_nvfp4_grouped")
    return out


def emulated_fp4_matmul(aq: QuantizedTensor, bq: QuantizedTensor, *, transpose_b: bool = False,
                        bf16_out: bool = False) -> torch.Tensor:
    """matmul(dequantize(aq), dequantize(bq)) with 32-bit accumulation
    (qlinear.py:74-93).  Returns a float32 CUDA tensor (bf16-rounded values
    when ``bf16_out``)."""
    if len(aq.shape) != 2 or len(bq.shape) != 2:
        raise InvalidInputError("emulated matmul is defined for 2-D operands")
    if transpose_b:
        if aq.shape[1] != bq.shape[1]:
            raise InvalidInputError(f"inner dimensions differ: {aq.shape} x {tuple(bq.shape[::-1])}")
        if bf16_out:
            return gemm_nvfp4(aq, bq, torch.bfloat16).to(torch.float32)
        return gemm_nvfp4(aq, bq, torch.float32)
    if aq.shape[1] != bq.shape[0]:
        raise InvalidInputError(f"inner dimensions differ: {aq.shape} x {bq.shape}")
    # the reference's own arithmetic: operands rounded once to float32, float32
    # products summed in ascending k (bit-identical to _accum_matmul_f32)
    A = dequantize_tensor(aq, torch.float32).contiguous()
    B = dequantize_tensor(bq, torch.float32).contiguous()
    M, K = A.shape
    N = B.shape[1]
    C = torch.empty((M, N), dtype=torch.float32, device=A.device)
    L = _lib.load()
    _lib.check(L.f46_matmul_f32_ordered(A.data_ptr(), B.data_ptr(), M, N, K, C.data_ptr(), _stream()),
               "f46_matmul_f32_ordered")
    return round_to_bf16(C) if bf16_out else C


def _quantize_1d(X, config, sr_tag: int = 0):
    """qlinear.py:96-99: 4/6 or fixed quantization along the last dim."""
    from .adaptive import quantize_tensor_adaptive
    from .blockquant import quantize_tensor

    if config.scale_mode == "adaptive":
        return quantize_tensor_adaptive(X, config, sr_tag=sr_tag)
    return quantize_tensor(X, config, sr_tag=sr_tag)


def _check_2d(name: str, t) -> None:
    if len(tuple(t.shape)) != 2:
        raise InvalidInputError(f"{name} must be 2-D")


def linear_forward(x, W, config, *, bf16_out: bool = False) -> torch.Tensor:
    """y = q(x) @ q(W)^T, both operands RNE (qlinear.py:107-120): x blocked 1-D
    along `in`, W in 16x16 tiles; the GEMM runs on tcgen05."""
    from dataclasses import replace

    from .transforms import quantize_weights_2d

    _check_2d("x", x)
    _check_2d("W", W)
    if x.shape[1] != W.shape[1]:
        raise InvalidInputError("x and W disagree on the input dimension")
    rne = replace(config, rounding="rne")
    xq = _quantize_1d(x, rne, sr_tag=0)
    wq = quantize_weights_2d(W, rne, with_transpose=False)
    return emulated_fp4_matmul(xq, wq, transpose_b=True, bf16_out=bf16_out)


def linear_dgrad(dy, W, config, *, bf16_out: bool = False) -> torch.Tensor:
    """dx = q(dy) @ q(W) (qlinear.py:123-135).  dy is blocked along `out`; W's
    16x16 tiles make W^T an NVFP4 tensor blocked along `out` too, so the
    product is a K-major (TN) tcgen05 GEMM against the transposed container."""
    from dataclasses import replace

    from .transforms import quantize_weights_2d

    _check_2d("dy", dy)
    _check_2d("W", W)
    if dy.shape[1] != W.shape[0]:
        raise InvalidInputError("dy and W disagree on the output dimension")
    dyq = _quantize_1d(dy, config, sr_tag=1)
    wq = quantize_weights_2d(W, replace(config, rounding="rne"))
    return emulated_fp4_matmul(dyq, wq.transposed, transpose_b=True, bf16_out=bf16_out)


def linear_wgrad(dy, x, config, *, bf16_out: bool = False) -> torch.Tensor:
    """dW = q(T dy)^T @ q(T x) (qlinear.py:138-159): both operands pass
    through the 16-wide randomized Hadamard transform along the batch axis
    (f46_rht16, float64), are quantized along it with the configured rounding
    (stochastic: numpy-exact Philox uniforms, tags 2 and 3), and meet in a
    K-major tcgen05 GEMM contracting over the batch."""
    from .blockquant import as_device_tensor
    from .transforms import RhtSpec, apply_rht

    _check_2d("dy", dy)
    _check_2d("x", x)
    if dy.shape[0] != x.shape[0]:
        raise InvalidInputError("dy and x disagree on the batch dimension")
    spec = RhtSpec(seed=config.seed)
    if dy.shape[0] % spec.size:
        raise InvalidInputError(f"batch dimension must be a multiple of {spec.size} for wgrad")
    a = apply_rht(as_device_tensor(dy).T.contiguous(), spec)  # (out, batch)
    b = apply_rht(as_device_tensor(x).T.contiguous(), spec)   # (in, batch)
    aq = _quantize_1d(a, config, sr_tag=2)
    bq = _quantize_1d(b, config, sr_tag=3)
    return emulated_fp4_matmul(aq, bq, transpose_b=True, bf16_out=bf16_out)
