"""NVFP4 block quantization on B200 behind the reference's API.

Mirrors fp4emu.blockquant (reference: /root/reference/pkg/src/fp4emu/
blockquant.py) name for name: ``QuantConfig`` (:68-140, validation kept
verbatim), ``QuantizedTensor`` (:156-188), ``compute_tensor_scale``
(:215-222), ``compute_block_scale`` (:225-236), ``quantize_tensor``
(:334-360), ``dequantize_tensor`` (:363-376), ``quantize_block`` (:379-414),
``reconstruction_mse`` (:485-489).

All arithmetic runs in libfouroversix.so (CUDA, sm_100a) through the C ABI of
include/fouroversix.h.  Inputs may be torch tensors (any device; CUDA
preferred) or numpy arrays; they are moved to the current CUDA device.  The
container keeps its payload on the GPU in the tensor-core layout (packed
E2M1 codes + E4M3 scales in the tcgen05 128x4 tiling + a device float64
alpha) and materialises the reference's host views (``codes``,
``scale_codes``, ``alpha``) lazily on first access.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, InvalidInputError

__all__ = [
    "NVFP4_BLOCK",
    "MXFP4_BLOCK",
    "QuantConfig",
    "BlockQuantResult",
    "QuantizedTensor",
    "compute_tensor_scale",
    "compute_block_scale",
    "quantize_block",
    "quantize_tensor",
    "dequantize_tensor",
    "reconstruction_mse",
    "sr_keys",
]

NVFP4_BLOCK = 16
MXFP4_BLOCK = 32

_FORMATS = ("nvfp4", "mxfp4")
_SCALE_MODES = ("fixed6", "fixed4", "adaptive")
_RULES = ("mse", "l1", "absmax")
_ROUNDINGS = ("rne", "sr")


@dataclass(frozen=True)
class QuantConfig:
    """Quantization settings (identical fields, defaults and validation to
    the reference, blockquant.py:68-140)."""

    fmt: str = "nvfp4"
    scale_mode: str = "fixed6"
    rule: str = "mse"
    rounding: str = "rne"
    seed: int = 0
    fp8_cap: Optional[float] = None
    sim_hp_scales: bool = False
    sim_hp_values: bool = False
    threshold: Optional[float] = None

    def __post_init__(self):
        if self.fmt not in _FORMATS:
            raise ConfigError(f"unknown format {self.fmt!r}")
        if self.scale_mode not in _SCALE_MODES:
            raise ConfigError(f"unknown scale_mode {self.scale_mode!r}")
        if self.rule not in _RULES:
            raise ConfigError(f"unknown rule {self.rule!r}")
        if self.rounding not in _ROUNDINGS:
            raise ConfigError(f"unknown rounding {self.rounding!r}")
        if not isinstance(self.seed, int) or self.seed < 0:
            raise ConfigError("seed must be a non-negative integer")
        if self.fmt == "mxfp4" and self.scale_mode != "fixed6":
            raise ConfigError("mxfp4 supports only scale_mode='fixed6'")
        cap = self.fp8_cap
        if self.scale_mode == "adaptive":
            if cap is None:
                cap = 256.0
            if cap != 256.0:
                raise ConfigError("adaptive mode requires fp8_cap == 256")
        else:
            if cap is None:
                cap = 448.0
            if cap not in (448.0, 256.0):
                raise ConfigError("fp8_cap must be 448 or 256")
        object.__setattr__(self, "fp8_cap", float(cap))
        if self.threshold is not None and not (0.0 <= self.threshold <= 6.0):
            raise InvalidInputError("threshold must lie in [0, 6]")

    @property
    def block_size(self) -> int:
        return NVFP4_BLOCK if self.fmt == "nvfp4" else MXFP4_BLOCK

    @property
    def m_tensor(self) -> float:
        return 4.0 if self.scale_mode == "fixed4" else 6.0

    def candidate_ms(self) -> tuple[float, ...]:
        if self.scale_mode == "fixed6":
            return (6.0,)
        if self.scale_mode == "fixed4":
            return (4.0,)
        return (6.0, 4.0)


@dataclass
class BlockQuantResult:
    """Outcome of quantizing one block (blockquant.py:143-153)."""

    codes: np.ndarray
    scale_code: int
    chosen_m: int
    err_mse: float
    err_l1: float
    err_max: float
    dequant: np.ndarray = field(repr=False, default=None)


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_02010_b200 needs a CUDA device (sm_100a); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_DT_OF = {torch.bfloat16: _lib.DT_BF16, torch.float32: _lib.DT_F32, torch.float64: _lib.DT_F64}


def as_device_tensor(X) -> torch.Tensor:
    """Move an array-like to the CUDA device in a dtype the kernels take.

    bf16 / f32 / f64 stay as they are; f16 and integers widen exactly
    (f16 -> f32, ints -> f64).  numpy float64 input stays float64, so the
    reference's own float64 test tensors are quantized with the reference's
    float64 semantics (the kernels' exact path).
    """
    dev = _device()
    if isinstance(X, torch.Tensor):
        t = X
    else:
        a = np.asarray(X)
        if a.dtype == np.float32:
            t = torch.from_numpy(np.ascontiguousarray(a))
        else:
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    if t.dtype == torch.float16:
        t = t.to(torch.float32)
    elif t.dtype not in _DT_OF:
        t = t.to(torch.float64)
    return t.to(dev, non_blocking=True).contiguous()


def _validated_shape(t: torch.Tensor):
    if t.dim() == 0:
        raise InvalidInputError("tensor must have at least one dimension")
    if t.numel() == 0:
        raise InvalidInputError("tensor must be non-empty")
    cols = t.shape[-1]
    return t.numel() // cols, cols


def scales_tc_bytes(rows: int, cols: int) -> int:
    nb = -(-cols // 16)
    return -(-rows // 128) * -(-nb // 4) * 512


def tc_to_rowmajor(scales_tc: torch.Tensor, rows: int, nb: int) -> torch.Tensor:
    """Gather the reference's [rows, nb] scale layout out of the tcgen05 tiling
    (include/fouroversix.h, offset(r, kb))."""
    dev = scales_tc.device
    r = torch.arange(rows, device=dev, dtype=torch.int64)[:, None]
    kb = torch.arange(nb, device=dev, dtype=torch.int64)[None, :]
    kb4 = -(-nb // 4)
    off = ((r // 128) * kb4 + kb // 4) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + kb % 4
    return scales_tc[off]


def rowmajor_to_tc(scales_rm: torch.Tensor, rows: int, nb: int) -> torch.Tensor:
    dev = scales_rm.device
    out = torch.zeros(scales_tc_bytes(rows, nb * 16), dtype=torch.uint8, device=dev)
    r = torch.arange(rows, device=dev, dtype=torch.int64)[:, None]
    kb = torch.arange(nb, device=dev, dtype=torch.int64)[None, :]
    kb4 = -(-nb // 4)
    off = ((r // 128) * kb4 + kb // 4) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + kb % 4
    out[off.reshape(-1)] = scales_rm.reshape(-1)
    return out


# ---------------------------------------------------------------------------
# container
# ---------------------------------------------------------------------------

class QuantizedTensor:
    """Quantized container (reference blockquant.py:156-188).

    Device payload (what the GEMM consumes):
      packed_codes  uint8 [rows, nb*8]  two E2M1 codes per byte, even element low
      scales_tc     uint8 tcgen05 128x4-tiled E4M3 scales
      alpha_dev     float64 [1] tensor scale
    Reference views (host numpy, materialised lazily): ``codes`` (one code per
    element, shape = source shape), ``scale_codes`` ([rows, nb]), ``alpha``.
    Constructing it with the reference's keyword arguments
    ``QuantizedTensor(shape=, fmt=, alpha=, scale_codes=, codes=)`` uploads
    them into the device layout.
    """

    def __init__(self, shape, fmt, alpha, scale_codes, codes):
        shape = tuple(int(s) for s in shape)
        self.shape = shape
        self.fmt = fmt
        cols = shape[-1] if len(shape) else 1
        rows = int(np.prod(shape[:-1], dtype=np.int64)) if len(shape) > 1 else 1
        nb = -(-cols // 16)
        dev = _device()
        sc = np.ascontiguousarray(np.asarray(scale_codes, dtype=np.uint8).reshape(rows, nb))
        c = np.asarray(codes, dtype=np.uint8).reshape(rows, cols)
        pad = np.zeros((rows, nb * 16), np.uint8)
        pad[:, :cols] = c & 0xF
        packed = (pad[:, 0::2] | (pad[:, 1::2] << 4)).astype(np.uint8)
        self.packed_codes = torch.from_numpy(packed).to(dev)
        self.scales_rm = torch.from_numpy(sc).to(dev)
        self.scales_tc = rowmajor_to_tc(self.scales_rm, rows, nb)
        self.alpha_dev = torch.tensor([float(alpha)], dtype=torch.float64, device=dev)
        self._alpha = float(alpha)
        self.pick4 = None

    @classmethod
    def _from_device(cls, shape, fmt, packed_codes, scales_tc, alpha_dev, scales_rm=None,
                     pick4=None, alpha=None):
        self = cls.__new__(cls)
        self.shape = tuple(int(s) for s in shape)
        self.fmt = fmt
        self.packed_codes = packed_codes
        self.scales_tc = scales_tc
        self.scales_rm = scales_rm
        self.alpha_dev = alpha_dev
        self._alpha = alpha
        self.pick4 = pick4
        return self

    # -- geometry ----------------------------------------------------------
    @property
    def rows(self) -> int:
        return int(np.prod(self.shape[:-1], dtype=np.int64)) if len(self.shape) > 1 else 1

    @property
    def cols(self) -> int:
        return self.shape[-1]

    @property
    def nblocks_per_row(self) -> int:
        return -(-self.cols // 16)

    @property
    def block_size(self) -> int:
        return NVFP4_BLOCK if self.fmt == "nvfp4" else MXFP4_BLOCK

    @property
    def num_blocks(self) -> int:
        return self.rows * self.nblocks_per_row

    # -- reference views -----------------------------------------------------
    @property
    def alpha(self) -> float:
        if self._alpha is None:
            self._alpha = float(self.alpha_dev.item())
        return self._alpha

    def scale_codes_device(self) -> torch.Tensor:
        if self.scales_rm is None:
            self.scales_rm = tc_to_rowmajor(self.scales_tc, self.rows, self.nblocks_per_row)
        return self.scales_rm

    @property
    def scale_codes(self) -> np.ndarray:
        return self.scale_codes_device().cpu().numpy()

    def codes_device(self) -> torch.Tensor:
        """Unpacked codes [rows, cols] on the device (one uint8 per element)."""
        p = self.packed_codes
        out = torch.stack([p & 0xF, p >> 4], dim=-1).reshape(self.rows, -1)
        return out[:, : self.cols]

    @property
    def codes(self) -> np.ndarray:
        return self.codes_device().cpu().numpy().reshape(self.shape)

    def __eq__(self, other) -> bool:
        if not isinstance(other, QuantizedTensor):
            return NotImplemented
        return (
            self.shape == other.shape
            and self.fmt == other.fmt
            and self.alpha == other.alpha
            and torch.equal(self.scale_codes_device(), other.scale_codes_device().to(self.scales_tc.device))
            and torch.equal(self.packed_codes, other.packed_codes.to(self.scales_tc.device))
        )

    def __repr__(self):
        return f"QuantizedTensor(shape={self.shape}, fmt={self.fmt!r}, device={self.scales_tc.device})"


# ---------------------------------------------------------------------------
# core launcher
# ---------------------------------------------------------------------------

def _raise_flags(flags: torch.Tensor):
    f = int(flags.item())
    if f & _lib.FLAG_NONFINITE:
        raise InvalidInputError("tensor must be finite")
    if f & _lib.FLAG_NAN_SCALE:
        raise InvalidInputError("container holds a NaN scale code")


def _check_alpha_override(alpha) -> float:
    a = float(alpha)
    if not np.isfinite(a) or a <= 0.0:
        raise InvalidInputError("alpha override must be positive and finite")
    return a


def amax_device(t: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """max|t| as a float64 [1] device tensor (K1); folds into `out` if given."""
    L = _lib.load()
    if out is None:
        out = torch.zeros(1, dtype=torch.float64, device=t.device)
    _lib.check(L.f46_amax(t.data_ptr(), _DT_OF[t.dtype], t.numel(), out.data_ptr(), _stream()),
               "f46_amax")
    return out


def sr_keys(seed: int, sr_tag: int) -> tuple[int, int, int, int]:
    """Philox4x64 keys of the reference's stochastic-rounding streams
    (blockquant.py:253-257): SeedSequence(seed, spawn_key=(tag, m)) for m = 6, 4."""
    k6 = np.random.SeedSequence(entropy=seed, spawn_key=(sr_tag, 6)).generate_state(2, np.uint64)
    k4 = np.random.SeedSequence(entropy=seed, spawn_key=(sr_tag, 4)).generate_state(2, np.uint64)
    return int(k6[0]), int(k6[1]), int(k4[0]), int(k4[1])


# tensors up to this size take the fused single-launch amax + quantize
FUSED_MAX_BYTES = int(__import__('os').environ.get('F46_FUSED_MAX_MB', '96')) << 20


def quantize_1d(X, mode: str, rule: str = "mse", fp8_cap: float = 448.0, alpha=None, *,
                d_amax: Optional[torch.Tensor] = None, check_finite: bool = True,
                want_rowmajor: bool = False, want_pick4: bool = False,
                rounding: str = "rne", seed: int = 0, sr_tag: int = 0) -> QuantizedTensor:
    """Quantize X (16-blocks along the last dim) with libfouroversix.

    mode  "fixed6" | "fixed4" | "adaptive";  alpha: override (float) or None.
    d_amax: a precomputed (e.g. all-reduced) device amax; else K1 runs here.
    rounding "sr" draws the reference's Philox uniforms (seed, sr_tag) on the GPU.
    """
    L = _lib.load()
    t = as_device_tensor(X)
    rows, cols = _validated_shape(t)
    dev = t.device
    nb = -(-cols // 16)
    m_tensor = 4.0 if mode == "fixed4" else 6.0
    mcap = m_tensor * (256.0 if mode == "adaptive" else float(fp8_cap))
    codes = torch.empty((rows, nb * 8), dtype=torch.uint8, device=dev)
    scales_tc = torch.empty(scales_tc_bytes(rows, cols), dtype=torch.uint8, device=dev)
    if cols % 64 != 0:
        scales_tc.zero_()
    scales_rm = torch.empty((rows, nb), dtype=torch.uint8, device=dev) if want_rowmajor else None
    pick4 = torch.empty((rows, nb), dtype=torch.uint8, device=dev) if want_pick4 else None
    alpha_dev = torch.empty(1, dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    a_over = 0.0
    if alpha is not None:
        a_over = _check_alpha_override(alpha)
    elif (d_amax is None and rounding == "rne" and scales_rm is None and pick4 is None
          and t.dtype != torch.float64 and t.numel() * t.element_size() <= FUSED_MAX_BYTES):
        # L2-sized tensor: amax and quantize in one cooperative launch (the
        # quantize pass re-reads its tiles from L2)
        work = torch.zeros(2, dtype=torch.float64, device=dev)
        rc = L.f46_quantize_fused(t.data_ptr(), _DT_OF[t.dtype], rows, cols, _lib.MODE[mode],
                                  _lib.RULE[rule], mcap, work.data_ptr(), codes.data_ptr(),
                                  scales_tc.data_ptr(), alpha_dev.data_ptr(), flags.data_ptr(),
                                  _stream())
        if rc == _lib.F46_OK:
            if check_finite:
                _raise_flags(flags)
            shape = tuple(X.shape) if hasattr(X, "shape") else tuple(t.shape)
            return QuantizedTensor._from_device(shape, "nvfp4", codes, scales_tc, alpha_dev)
        if rc != _lib.F46_ERR_UNSUPPORTED:
            _lib.check(rc, "f46_quantize_fused")
        d_amax = amax_device(t)
    elif d_amax is None:
        d_amax = amax_device(t)
    if rounding == "sr":
        k = sr_keys(seed, sr_tag)
        rc = L.f46_quantize_sr(
            t.data_ptr(), _DT_OF[t.dtype], rows, cols, _lib.MODE[mode], _lib.RULE[rule], mcap,
            _lib.ptr(d_amax), a_over, k[0], k[1], k[2], k[3], codes.data_ptr(),
            scales_tc.data_ptr(), _lib.ptr(scales_rm), _lib.ptr(pick4), alpha_dev.data_ptr(),
            flags.data_ptr(), _stream())
        _lib.check(rc, "f46_quantize_sr")
    else:
        rc = L.f46_quantize(
            t.data_ptr(), _DT_OF[t.dtype], rows, cols, _lib.MODE[mode], _lib.RULE[rule], mcap,
            _lib.ptr(d_amax), a_over, codes.data_ptr(), scales_tc.data_ptr(), _lib.ptr(scales_rm),
            _lib.ptr(pick4), alpha_dev.data_ptr(), flags.data_ptr(), _stream())
        _lib.check(rc, "f46_quantize")
    if check_finite:
        _raise_flags(flags)
    shape = tuple(X.shape) if hasattr(X, "shape") else tuple(t.shape)
    return QuantizedTensor._from_device(shape, "nvfp4", codes, scales_tc, alpha_dev,
                                        scales_rm=scales_rm, pick4=pick4,
                                        alpha=(a_over if alpha is not None else None))


# ---------------------------------------------------------------------------
# public API (reference names)
# ---------------------------------------------------------------------------

def compute_tensor_scale(X, m_fp4: float, fp8_cap: float) -> float:
    """alpha = max|X| / (m_fp4 * fp8_cap) through float32; 1.0 if all zero
    (blockquant.py:215-222).  The max runs on the GPU (K1)."""
    t = as_device_tensor(X)
    _validated_shape(t)
    amax = float(amax_device(t).item())
    if not np.isfinite(amax):
        raise InvalidInputError("tensor must be finite")
    if amax == 0.0:
        return 1.0
    return float(np.float32(amax) / np.float32(m_fp4 * fp8_cap))


def _require_plain_nvfp4(config: QuantConfig):
    if config.fmt != "nvfp4":
        raise ConfigError("the B200 path implements the nvfp4 format (mxfp4 is out of scope)")


def quantize_tensor(X, config: QuantConfig, alpha: Optional[float] = None, sr_tag: int = 0,
                    **kw) -> QuantizedTensor:
    """Fixed-target (6 or 4) NVFP4 quantization (blockquant.py:334-360)."""
    if config.scale_mode == "adaptive":
        raise ConfigError("use quantize_tensor_adaptive for adaptive mode")
    if config.sim_hp_scales or config.sim_hp_values or config.threshold is not None:
        raise ConfigError("simulation knobs require quantize_tensor_simulated")
    _require_plain_nvfp4(config)
    return quantize_1d(X, config.scale_mode, config.rule, config.fp8_cap, alpha,
                       rounding=config.rounding, seed=config.seed, sr_tag=sr_tag, **kw)


def dequantize_tensor(q: QuantizedTensor, dtype: torch.dtype = torch.float64,
                      check: bool = True) -> torch.Tensor:
    """decode(code) * alpha * decode(scale) on the GPU (blockquant.py:363-376).

    The default float64 output is the reference's exact value (its return
    dtype); float32 / bfloat16 are that value rounded once (the fast paths).
    Returns a CUDA tensor of the container's shape.
    """
    L = _lib.load()
    if q.fmt != "nvfp4":
        raise ConfigError("the B200 path implements the nvfp4 format")
    dev = q.scales_tc.device
    out_dt = {torch.float32: _lib.DT_F32, torch.bfloat16: _lib.DT_BF16, torch.float64: _lib.DT_F64}[dtype]
    out = torch.empty((q.rows, q.cols), dtype=dtype, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = L.f46_dequantize(q.packed_codes.data_ptr(), q.scales_tc.data_ptr(), _lib.SCALES_TC,
                          q.alpha_dev.data_ptr(), q.rows, q.cols, out.data_ptr(), out_dt,
                          flags.data_ptr(), _stream())
    _lib.check(rc, "f46_dequantize")
    if check:
        _raise_flags(flags)
    return out.reshape(q.shape)


def _block_input(block) -> torch.Tensor:
    """A block for the block-level API as a torch tensor where it already is
    (host or device): validation runs before anything is launched; the values
    move to the device in _block_ref."""
    if isinstance(block, torch.Tensor):
        return block
    return torch.from_numpy(np.ascontiguousarray(np.asarray(block, dtype=np.float64)))


def _block_ref(arr: torch.Tensor, alpha: float, m: float, u=None):
    """One block through f46_quantize_block_ref: the reference's float64
    single-block arithmetic (any length, any m) on the device.  Returns
    (codes, scale_code, sum diff^2, sum |diff|, max |diff|, dequant)."""
    L = _lib.load()
    x = as_device_tensor(arr.reshape(-1).to(torch.float64)).contiguous()
    n = x.numel()
    dev = x.device
    ud = None
    if u is not None:
        ud = as_device_tensor(np.asarray(u, dtype=np.float64).reshape(-1)).to(dev).contiguous()
    codes = torch.empty(n, dtype=torch.uint8, device=dev)
    work = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.empty(4, dtype=torch.float64, device=dev)
    rc = L.f46_quantize_block_ref(x.data_ptr(), n, float(alpha), float(m), _lib.ptr(ud),
                                  codes.data_ptr(), work.data_ptr(), out.data_ptr(), _stream())
    _lib.check(rc, "f46_quantize_block_ref")
    o = out.cpu().numpy()
    return codes.cpu().numpy(), int(o[0]), float(o[1]), float(o[2]), float(o[3]), work.cpu().numpy()


def compute_block_scale(block, alpha: float, m: float) -> np.uint8:
    """E4M3 code of max|block| / (alpha*m); zero blocks get code 1
    (blockquant.py:225-236); any block length and target m."""
    arr = _block_input(block).reshape(-1)
    if not bool(torch.isfinite(arr).all()):
        raise InvalidInputError("block must be finite")
    if alpha <= 0 or not np.isfinite(alpha):
        raise InvalidInputError("alpha must be positive and finite")
    if arr.numel() == 0:
        return np.uint8(1)
    return np.uint8(_block_ref(arr, alpha, m)[1])


def _block_result(arr: torch.Tensor, alpha: float, m: float, u=None) -> BlockQuantResult:
    codes, sc, ssq, sab, smx, deq = _block_ref(arr, alpha, m, u)
    n = arr.numel()
    return BlockQuantResult(codes=codes, scale_code=sc, chosen_m=int(m), err_mse=ssq / n,
                            err_l1=sab / n, err_max=smx, dequant=deq)


def _check_uniforms(u, n: int, what: str):
    if u is None:
        raise InvalidInputError(f"stochastic rounding requires uniforms{what}")
    if np.asarray(u).size != n:
        raise InvalidInputError("u must match the block length" if what == " u" else
                                "uniforms must match the block length")


def quantize_block(block, alpha: float, m: float, rounding: str = "rne", u=None) -> BlockQuantResult:
    """Quantize one block (any length) at a fixed target m (blockquant.py:379-414);
    stochastic rounding takes the explicit uniforms u."""
    arr = _block_input(block)
    if arr.dim() != 1 or arr.numel() == 0:
        raise InvalidInputError("block must be a non-empty 1-D array")
    if not bool(torch.isfinite(arr).all()):
        raise InvalidInputError("block must be finite")
    if rounding not in _ROUNDINGS:
        raise ConfigError(f"unknown rounding {rounding!r}")
    if rounding == "sr":
        _check_uniforms(u, arr.numel(), " u")
    return _block_result(arr, alpha, m, u if rounding == "sr" else None)


def reconstruction_mse(X, D) -> float:
    """Mean squared reconstruction error (blockquant.py:485-489), on the GPU in float64."""
    x = as_device_tensor(X).to(torch.float64)
    d = as_device_tensor(D).to(torch.float64)
    diff = d - x
    return float(torch.mean(diff * diff))
