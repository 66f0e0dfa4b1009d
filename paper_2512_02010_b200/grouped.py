"""Grouped (one tensor per MoE expert) quantization for the config-5 recipe.

The reference quantizes one tensor at a time; an expert-parallel MoE layer
holds E independent tensors per GPU, each with its
own tensor scale.  These entry points quantize all E in one launch each and
return the operands packed back to back -- the layout
``qlinear.gemm_nvfp4_grouped`` consumes -- with results identical to calling
the single-tensor function per expert (the reference semantics, one
``compute_tensor_scale`` per tensor, blockquant.py:215-222):

* ``quantize_grouped``          quantize_tensor[_adaptive] per expert (X, dY)
* ``quantize_weights_2d_grouped`` quantize_weights_2d per expert (W and W^T)
* ``quantize_wgrad_operand_grouped``  the WGRAD operand of linear_wgrad
  (reference qlinear.py:150-157): apply_rht(a.T, spec) then 1-D quantization
  along the token axis, fused into one transpose+RHT+quantize pass (f46_rht.cu)

All work is on the device through the C ABI; nothing here touches the host
beyond argument checks (no CPU fallback).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .blockquant import (QuantConfig, QuantizedTensor, _DT_OF, _raise_flags, _stream,
                         as_device_tensor, scales_tc_bytes)
from .errors import ConfigError, InvalidInputError
from .transforms import RhtSpec

__all__ = ["GroupedQuantized", "quantize_grouped", "quantize_weights_2d_grouped",
           "quantize_wgrad_operand_grouped"]


@dataclass
class GroupedQuantized:
    """E quantized [rows, cols] tensors back to back.

    codes     uint8 [E, rows, nb*8]   (nb = ceil(cols/16))
    scales_tc uint8 [E, scales_tc_bytes(rows, cols)]
    alpha_dev float64 [E]             per-expert tensor scale
    transposed  the [cols, rows] operands (2-D tile weights only)
    """

    shape: tuple
    codes: torch.Tensor
    scales_tc: torch.Tensor
    alpha_dev: torch.Tensor
    transposed: Optional["GroupedQuantized"] = None

    @property
    def groups(self) -> int:
        return self.codes.shape[0]

    def operands(self):
        """(codes, scales, alpha) as gemm_nvfp4_grouped takes them."""
        return self.codes, self.scales_tc, self.alpha_dev

    def group(self, e: int) -> QuantizedTensor:
        """Expert e as a QuantizedTensor (views, no copy)."""
        return QuantizedTensor._from_device(self.shape, "nvfp4", self.codes[e], self.scales_tc[e],
                                            self.alpha_dev[e:e + 1])


def _mcap(config: QuantConfig) -> float:
    return float(config.m_tensor) * float(config.fp8_cap)


def _check_config(config: QuantConfig):
    if config.fmt != "nvfp4":
        raise ConfigError("grouped quantization is defined for nvfp4")
    if config.rounding != "rne":
        raise ConfigError("grouped quantization implements rounding='rne'")
    if config.sim_hp_scales or config.sim_hp_values or config.threshold is not None:
        raise ConfigError("simulation knobs are not part of the B200 path")


def _as_groups(X, ndim: int = 3) -> torch.Tensor:
    t = as_device_tensor(X)
    if t.dim() != ndim:
        raise InvalidInputError(f"grouped input must be {ndim}-D [experts, ...]")
    if t.numel() == 0:
        raise InvalidInputError("tensor must be non-empty")
    if t.dtype not in (torch.bfloat16, torch.float32):
        raise InvalidInputError("grouped quantization takes BF16 or FP32 input")
    return t.contiguous()


def _empty(E, rows, cols, dev, zero_scales=False):
    nb = -(-cols // 16)
    codes = torch.empty((E, rows, nb * 8), dtype=torch.uint8, device=dev)
    mk = torch.zeros if zero_scales else torch.empty
    scales = mk((E, scales_tc_bytes(rows, cols)), dtype=torch.uint8, device=dev)
    return codes, scales


def _amax_grouped(t: torch.Tensor, n: int) -> torch.Tensor:
    L = _lib.load()
    E = t.shape[0]
    amax = torch.zeros(E, dtype=torch.float64, device=t.device)
    _lib.check(L.f46_amax_grouped(t.data_ptr(), _DT_OF[t.dtype], E, n, amax.data_ptr(), _stream()),
               "f46_amax_grouped")
    return amax


def quantize_grouped(X, config: QuantConfig, *, check_finite: bool = True) -> GroupedQuantized:
    """X [E, rows, cols]: each expert quantized along its last dim with its own
    tensor scale, as ``quantize_tensor_adaptive(X[e], config)`` (adaptive.py:83)
    or ``quantize_tensor(X[e], config)`` (blockquant.py:334) would."""
    _check_config(config)
    t = _as_groups(X)
    E, rows, cols = t.shape
    L = _lib.load()
    amax = _amax_grouped(t, rows * cols)
    codes, scales = _empty(E, rows, cols, t.device)
    alpha = torch.empty(E, dtype=torch.float64, device=t.device)
    flags = torch.zeros(1, dtype=torch.int32, device=t.device)
    rc = L.f46_quantize_grouped(t.data_ptr(), _DT_OF[t.dtype], E, rows, cols,
                                _lib.MODE[config.scale_mode], _lib.RULE[config.rule], _mcap(config),
                                amax.data_ptr(), codes.data_ptr(), scales.data_ptr(), alpha.data_ptr(),
                                flags.data_ptr(), _stream())
    _lib.check(rc, "f46_quantize_grouped")
    if check_finite:
        _raise_flags(flags)
    return GroupedQuantized((rows, cols), codes, scales, alpha)


def quantize_weights_2d_grouped(W, config: QuantConfig, *, with_transpose: bool = True,
                                check_finite: bool = True) -> GroupedQuantized:
    """W [E, R, C]: ``quantize_weights_2d(W[e], config)`` per expert
    (transforms.py:134-179), W and W^T from one pass."""
    _check_config(config)
    t = _as_groups(W)
    E, R, C = t.shape
    L = _lib.load()
    amax = _amax_grouped(t, R * C)
    codes, scales = _empty(E, R, C, t.device, zero_scales=True)
    codes_t, scales_t = _empty(E, C, R, t.device, zero_scales=True) if with_transpose else (None, None)
    alpha = torch.empty(E, dtype=torch.float64, device=t.device)
    flags = torch.zeros(1, dtype=torch.int32, device=t.device)
    rc = L.f46_quantize_2d_grouped(t.data_ptr(), _DT_OF[t.dtype], E, R, C,
                                   _lib.MODE[config.scale_mode], _lib.RULE[config.rule],
                                   _mcap(config), amax.data_ptr(), codes.data_ptr(),
                                   scales.data_ptr(), _lib.ptr(codes_t), _lib.ptr(scales_t),
                                   alpha.data_ptr(), flags.data_ptr(), _stream())
    _lib.check(rc, "f46_quantize_2d_grouped")
    if check_finite:
        _raise_flags(flags)
    q = GroupedQuantized((R, C), codes, scales, alpha)
    if with_transpose:
        q.transposed = GroupedQuantized((C, R), codes_t, scales_t, alpha)
    return q


def sign_mask(spec: RhtSpec) -> int:
    """Bit i set where the RHT diagonal's sign i is -1."""
    if spec.size != 16:
        raise ConfigError("the B200 transform kernel is the 16-wide one")
    return int(sum(1 << i for i, s in enumerate(np.asarray(spec.signs)) if s < 0))


def quantize_wgrad_operand_grouped(A, config: QuantConfig, spec: Optional[RhtSpec] = None, *,
                                   check_finite: bool = True) -> GroupedQuantized:
    """A [E, T, H] (tokens x features): per expert the WGRAD operand of
    ``linear_wgrad`` (reference qlinear.py:150-157) -- apply_rht(A[e].T, spec)
    quantized along the token axis -- as an [H, T] container, in one fused
    transpose + RHT + quantize pass per expert."""
    _check_config(config)
    spec = spec if spec is not None else RhtSpec(seed=config.seed)
    t = _as_groups(A)
    E, T, H = t.shape
    if T % spec.size:
        raise InvalidInputError(f"batch dimension must be a multiple of {spec.size} for wgrad")
    L = _lib.load()
    mask = sign_mask(spec)
    amax = torch.zeros(E, dtype=torch.float64, device=t.device)
    dt = _DT_OF[t.dtype]
    _lib.check(L.f46_rht_t_amax_grouped(t.data_ptr(), dt, E, T, H, mask, amax.data_ptr(), _stream()),
               "f46_rht_t_amax_grouped")
    codes, scales = _empty(E, H, T, t.device, zero_scales=True)
    alpha = torch.empty(E, dtype=torch.float64, device=t.device)
    flags = torch.zeros(1, dtype=torch.int32, device=t.device)
    rc = L.f46_quantize_rht_t_grouped(t.data_ptr(), dt, E, T, H, mask,
                                      _lib.MODE[config.scale_mode], _lib.RULE[config.rule],
                                      _mcap(config), amax.data_ptr(), codes.data_ptr(),
                                      scales.data_ptr(), alpha.data_ptr(), flags.data_ptr(), _stream())
    _lib.check(rc, "f46_quantize_rht_t_grouped")
    if check_finite:
        _raise_flags(flags)
    return GroupedQuantized((H, T), codes, scales, alpha)
