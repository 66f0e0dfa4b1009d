"""Four Over Six: per-block adaptive choice between block-max targets 6 and 4.

Mirrors fp4emu.adaptive (reference adaptive.py): ``quantize_tensor_adaptive``
(:83-101), ``quantize_block_adaptive`` (:104-146), ``selection_stats``
(:159-187).  Both candidates, the strict-'<' MSE selection with ties keeping
6, and the 256 tensor-scale cap are computed inside the fused sm_100a kernel
(f46_quantize, mode F46_ADAPTIVE); the choice is not stored in the container.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .blockquant import (
    BlockQuantResult,
    QuantConfig,
    QuantizedTensor,
    _block_result,
    _require_plain_nvfp4,
    as_device_tensor,
    dequantize_tensor,
    quantize_1d,
)
from .errors import ConfigError, InvalidInputError

__all__ = [
    "quantize_block_adaptive",
    "quantize_tensor_adaptive",
    "SelectionStats",
    "selection_stats",
]

_RULE_INDEX = {"mse": 0, "l1": 1, "absmax": 2}


def _require_adaptive(config: QuantConfig):
    if config.fmt != "nvfp4":
        raise ConfigError("adaptive mode requires the nvfp4 format")
    if config.scale_mode != "adaptive":
        raise ConfigError("config.scale_mode must be 'adaptive'")
    if config.sim_hp_scales or config.sim_hp_values or config.threshold is not None:
        raise ConfigError("simulation knobs require quantize_tensor_simulated")


def quantize_tensor_adaptive(X, config: QuantConfig, alpha: Optional[float] = None,
                             sr_tag: int = 0, **kw) -> QuantizedTensor:
    """Adaptively quantized container (adaptive.py:83-101).

    Extra keywords (B200 path): ``check_finite`` (default True: one device
    sync to raise InvalidInputError on non-finite input, as the reference
    does), ``d_amax`` (a precomputed, e.g. all-reduced, device amax),
    ``want_rowmajor`` / ``want_pick4`` (parity views).
    """
    _require_adaptive(config)
    _require_plain_nvfp4(config)
    return quantize_1d(X, "adaptive", config.rule, 256.0, alpha, rounding=config.rounding,
                       seed=config.seed, sr_tag=sr_tag, **kw)


def quantize_block_adaptive(block, alpha: float, rule: str = "mse", rounding: str = "rne",
                            u6=None, u4=None) -> BlockQuantResult:
    """Adaptive quantization of one block of any length (adaptive.py:104-146):
    both candidates in the reference's float64 arithmetic on the device, the
    rule's error compared with a strict '<' (ties keep 6)."""
    from .blockquant import _block_input, _block_result, _check_uniforms

    if rule not in _RULE_INDEX:
        raise ConfigError(f"unknown rule {rule!r}")
    arr = _block_input(block)
    if arr.dim() != 1 or arr.numel() == 0:
        raise InvalidInputError("block must be a non-empty 1-D array")
    if not bool(torch.isfinite(arr).all()):
        raise InvalidInputError("block must be finite")
    if rounding == "sr":  # both candidates' uniforms, before any launch
        _check_uniforms(u6, arr.numel(), "")
        _check_uniforms(u4, arr.numel(), "")
    cand = {m: _block_result(arr, alpha, m, u if rounding == "sr" else None)
            for m, u in ((6.0, u6), (4.0, u4))}
    key = {"mse": "err_mse", "l1": "err_l1", "absmax": "err_max"}[rule]
    return cand[4.0] if getattr(cand[4.0], key) < getattr(cand[6.0], key) else cand[6.0]


@dataclass
class SelectionStats:
    """How often each rule prefers the 4 target, and at what cost (adaptive.py:149-156)."""

    n_blocks: int
    fraction_4: dict
    disagreements: dict
    aggregate_mse: dict


def selection_stats(X, config: QuantConfig, alpha: Optional[float] = None,
                    sr_tag: int = 0) -> SelectionStats:
    """Per-rule selection statistics (adaptive.py:159-187) from one fused
    device pass (f46_selection_stats: exact float64 errors of both candidates,
    all three rules' picks, counts and chosen squared errors per block).
    fraction_4 and disagreements are exact counts; aggregate_mse sums the exact
    per-block errors in a fixed device order (per thread, then per CTA part,
    then the parts), so it equals the reference's numpy sum to float64
    rounding, not bit for bit."""
    from . import _lib
    from .blockquant import _DT_OF, _check_alpha_override, _stream, _validated_shape, amax_device

    _require_adaptive(config)
    _require_plain_nvfp4(config)
    if config.rounding != "rne":
        raise ConfigError("selection_stats on the B200 path uses rounding='rne'")
    L = _lib.load()
    t = as_device_tensor(X)
    rows, cols = _validated_shape(t)
    a_over, d_amax = 0.0, None
    # the reference validates X before anything else (_validated, blockquant.py:191-199):
    # one device max|X| doubles as the finiteness check, with or without an override
    d_amax = amax_device(t)
    if not bool(torch.isfinite(d_amax).all()):
        raise InvalidInputError("tensor must be finite")
    if alpha is not None:
        a_over = _check_alpha_override(alpha)
        d_amax = None
    nparts = 4 * torch.cuda.get_device_properties(t.device).multi_processor_count
    parts = torch.empty((nparts, 9), dtype=torch.float64, device=t.device)
    rc = L.f46_selection_stats(t.data_ptr(), _DT_OF[t.dtype], rows, cols, 1536.0,
                               _lib.ptr(d_amax), a_over, parts.data_ptr(), nparts, None, _stream())
    _lib.check(rc, "f46_selection_stats")
    tot = parts.sum(dim=0).cpu().numpy()
    n_blocks = rows * (-(-cols // 16))
    rules = ("mse", "l1", "absmax")
    frac = {r: float(tot[i]) / n_blocks for i, r in enumerate(rules)}
    dis = {"mse_vs_l1": int(tot[3]), "mse_vs_absmax": int(tot[4]), "l1_vs_absmax": int(tot[5])}
    agg = {r: float(tot[6 + i]) / (rows * cols) for i, r in enumerate(rules)}
    return SelectionStats(n_blocks=n_blocks, fraction_4=frac, disagreements=dis, aggregate_mse=agg)
