"""2-D 16x16-tile weight quantization (reference transforms.py:108-179).

``quantize_weights_2d`` mirrors the reference: one E4M3 scale per 16x16 tile,
chosen (fixed6 / fixed4 / adaptive 4/6 over all 256 values) by the
``f46_quantize_2d`` kernel in exact float64 with numpy's pairwise error-sum
order.  Because the tile scale is shared by the tile's rows and columns, the
same pass also yields W^T as an NVFP4 tensor blocked along W's rows; it is
attached as ``q.transposed`` and is what ``linear_dgrad``'s GEMM consumes
(qlinear.py:123-135: dy @ W needs W blocked along `out`).

``RhtSpec`` / ``apply_rht`` / ``invert_rht`` mirror the randomized Hadamard
transform of the gradient recipe (transforms.py:41-105): the sign diagonal is
drawn on the host exactly as the reference draws it (numpy Philox from
SeedSequence(seed, spawn_key=(0x5D,)) -- a 16-entry parameter), and the
transform itself runs in the f46_rht16 kernel in float64 with numpy's
butterfly order, so its output is bit-identical to the reference's.
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

__all__ = ["TILE", "RhtSpec", "apply_rht", "invert_rht", "quantize_weights_2d"]

TILE = 16
_SIGN_TAG = 0x5D  # transforms.py:38


class RhtSpec:
    """Transform parameters (transforms.py:44-67); signs derive from the seed
    unless given."""

    def __init__(self, size: int = 16, seed: int = 0, signs=None):
        if size < 1 or size & (size - 1):
            raise ConfigError("transform size must be a power of two")
        self.size = size
        self.seed = seed
        if signs is None:
            ss = np.random.SeedSequence(entropy=seed, spawn_key=(_SIGN_TAG,))
            rng = np.random.Generator(np.random.Philox(ss))
            signs = rng.integers(0, 2, size=size) * 2.0 - 1.0
        else:
            signs = np.asarray(signs, dtype=np.float64)
            if signs.shape != (size,) or not np.isin(signs, (-1.0, 1.0)).all():
                raise ConfigError("signs must be +-1 and match size")
        self.signs = np.ascontiguousarray(signs, dtype=np.float64)


def _rht_kernel(t: torch.Tensor, signs: np.ndarray) -> torch.Tensor:
    L = _lib.load()
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    sg = np.ascontiguousarray(signs, dtype=np.float64)
    rc = L.f46_rht16(t.data_ptr(), _DT_OF[t.dtype], t.numel(), sg.ctypes.data, out.data_ptr(),
                     _stream())
    _lib.check(rc, "f46_rht16")
    return out


def _grouped(X, size: int) -> torch.Tensor:
    t = as_device_tensor(X)
    if t.dim() == 0 or t.shape[-1] % size:
        raise InvalidInputError(f"last dimension must be a positive multiple of {size}")
    if size != 16:
        raise ConfigError("the B200 transform kernel is the 16-wide one")
    return t.contiguous()


def apply_rht(X, spec: RhtSpec) -> torch.Tensor:
    """y = fwht(g * signs) / sqrt(16) per group of 16 along the last dim
    (transforms.py:92-97); float64 CUDA tensor."""
    return _rht_kernel(_grouped(X, spec.size), spec.signs)


def invert_rht(Y, spec: RhtSpec) -> torch.Tensor:
    """x = (fwht(g) / sqrt(16)) * signs (transforms.py:100-105)."""
    t = _grouped(Y, spec.size)
    y = _rht_kernel(t, np.ones(spec.size))
    sg = torch.from_numpy(spec.signs).to(y.device)
    return (y.reshape(-1, spec.size) * sg).reshape(y.shape)


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
