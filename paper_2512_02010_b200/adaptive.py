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
    return quantize_1d(X, "adaptive", config.rule, 256.0, alpha, **kw)


def quantize_block_adaptive(block, alpha: float, rule: str = "mse", rounding: str = "rne",
                            u6=None, u4=None) -> BlockQuantResult:
    """Adaptive quantization of one block of <= 16 values (adaptive.py:104-146)."""
    if rule not in _RULE_INDEX:
        raise ConfigError(f"unknown rule {rule!r}")
    arr = as_device_tensor(block)
    if arr.dim() != 1 or arr.numel() == 0:
        raise InvalidInputError("block must be a non-empty 1-D array")
    if not bool(torch.isfinite(arr).all()):
        raise InvalidInputError("block must be finite")
    if rounding == "sr":
        if u6 is None or u4 is None:
            raise InvalidInputError("stochastic rounding requires uniforms")
        raise ConfigError("stochastic rounding is not implemented on the B200 path yet")
    if arr.numel() > 16:
        raise InvalidInputError("the B200 path quantizes 16-element NVFP4 blocks")
    q = quantize_1d(arr.reshape(1, -1), "adaptive", rule, 256.0, alpha, want_pick4=True)
    m = 4 if int(q.pick4[0, 0].item()) else 6
    return _block_result(arr, q, m)


@dataclass
class SelectionStats:
    """How often each rule prefers the 4 target, and at what cost (adaptive.py:149-156)."""

    n_blocks: int
    fraction_4: dict
    disagreements: dict
    aggregate_mse: dict


def selection_stats(X, config: QuantConfig, alpha: Optional[float] = None,
                    sr_tag: int = 0) -> SelectionStats:
    """Per-rule selection statistics (adaptive.py:159-187), from three fused
    device passes (one per rule) and float64 device reductions."""
    _require_adaptive(config)
    _require_plain_nvfp4(config)
    t = as_device_tensor(X)
    picks, agg = {}, {}
    a = alpha
    for rule in _RULE_INDEX:
        q = quantize_1d(t, "adaptive", rule, 256.0, a, want_pick4=True)
        a = q.alpha if a is None else a
        picks[rule] = q.pick4.bool()
        d = dequantize_tensor(q, torch.float64).reshape(-1) - t.reshape(-1).to(torch.float64)
        agg[rule] = float(torch.sum(d * d) / t.numel())
    n_blocks = int(picks["mse"].numel())
    frac = {r: float(p.float().mean()) for r, p in picks.items()}
    pairs = (("mse", "l1"), ("mse", "absmax"), ("l1", "absmax"))
    dis = {f"{a_}_vs_{b_}": int((picks[a_] != picks[b_]).sum()) for a_, b_ in pairs}
    return SelectionStats(n_blocks=n_blocks, fraction_4=frac, disagreements=dis, aggregate_mse=agg)
