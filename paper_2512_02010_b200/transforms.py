"""2-D 16x16-tile weight quantization (reference transforms.py:108-179).

``quantize_weights_2d`` mirrors the reference: one E4M3 scale per 16x16 tile,
chosen (fixed6 / fixed4 / adaptive 4/6 over all 256 values) by the
``f46_quantize_2d`` kernel in exact float64 with numpy's pairwise error-sum
order.  Because the tile scale is shared by the tile's rows and columns, the
same pass also yields W^T as an NVFP4 tensor blocked along W's rows; it is
attached as ``q.transposed`` and is what ``linear_dgrad``'s GEMM consumes
(qlinear.py:123-135: dy @ W needs W blocked along `out`).

The randomized Hadamard transform (transforms.py:41-105) belongs to the
gradient recipe and is not on the B200 path yet.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib
from .blockquant import (
    QuantConfig,
    QuantizedTensor,
    _DT_OF,
    _check_alpha_override,
    _raise_flags,
    _stream,
    amax_device,
    as_device_tensor,
    scales_tc_bytes,
)
from .errors import ConfigError, InvalidInputError

__all__ = ["TILE", "quantize_weights_2d"]

TILE = 16


def quantize_weights_2d(W, config: QuantConfig, alpha: Optional[float] = None, sr_tag: int = 0,
                        *, with_transpose: bool = True, check_finite: bool = True,
                        want_rowmajor: bool = False) -> QuantizedTensor:
    """Quantize a 2-D weight with one scale per 16x16 tile (transforms.py:134-179)."""
    if config.fmt != "nvfp4":
        raise ConfigError("2-D tile quantization is defined for nvfp4")
    if config.rounding != "rne":
        raise ConfigError("the B200 path implements rounding='rne' (stochastic rounding is a "
                          "later row of the build plan)")
    if config.sim_hp_scales or config.sim_hp_values or config.threshold is not None:
        raise ConfigError("simulation knobs are not part of the B200 path")
    L = _lib.load()
    t = as_device_tensor(W)
    if t.dim() != 2:
        raise InvalidInputError("weights must be 2-D")
    if t.numel() == 0:
        raise InvalidInputError("tensor must be non-empty")
    R, C = t.shape
    dev = t.device
    mode = config.scale_mode
    mcap = (4.0 if mode == "fixed4" else 6.0) * float(config.fp8_cap)
    nbc, nbr = -(-C // TILE), -(-R // TILE)
    codes = torch.empty((R, nbc * 8), dtype=torch.uint8, device=dev)
    scales_tc = torch.zeros(scales_tc_bytes(R, C), dtype=torch.uint8, device=dev)
    scales_rm = torch.empty((R, nbc), dtype=torch.uint8, device=dev) if want_rowmajor else None
    codes_t = torch.empty((C, nbr * 8), dtype=torch.uint8, device=dev) if with_transpose else None
    scales_tc_t = (torch.zeros(scales_tc_bytes(C, R), dtype=torch.uint8, device=dev)
                   if with_transpose else None)
    alpha_dev = torch.empty(1, dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    a_over, d_amax = 0.0, None
    if alpha is not None:
        a_over = _check_alpha_override(alpha)
    else:
        d_amax = amax_device(t)
    rc = L.f46_quantize_2d(
        t.data_ptr(), _DT_OF[t.dtype], R, C, _lib.MODE[mode], _lib.RULE[config.rule], mcap,
        _lib.ptr(d_amax), a_over, codes.data_ptr(), scales_tc.data_ptr(), _lib.ptr(scales_rm),
        None, _lib.ptr(codes_t), _lib.ptr(scales_tc_t), alpha_dev.data_ptr(), flags.data_ptr(),
        _stream())
    _lib.check(rc, "f46_quantize_2d")
    if check_finite:
        _raise_flags(flags)
    known = a_over if alpha is not None else None
    q = QuantizedTensor._from_device((R, C), "nvfp4", codes, scales_tc, alpha_dev,
                                     scales_rm=scales_rm, alpha=known)
    q.transposed = (QuantizedTensor._from_device((C, R), "nvfp4", codes_t, scales_tc_t, alpha_dev,
                                                 alpha=known) if with_transpose else None)
    return q
