"""ctypes front end of the CPU oracle (fouroversix_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference leg of bench.py, always as the checker, never
as the thing measured for the GPU arm.  The product package
(paper_2512_02010_b200) never imports this module.

Every function restates the reference's float64 semantics (see the C file's
header for the file:line map into /root/reference/pkg/src/fp4emu).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle46.so")

DT_F32, DT_BF16, DT_F64 = 0, 1, 2
MODES = {"fixed6": 0, "fixed4": 1, "adaptive": 2}
RULES = {"mse": 0, "l1": 1, "absmax": 2}

_lib = None


def build() -> str:
    """Compile the oracle with its own Makefile (no reference sources used)."""
    subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        c_p = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.fo_quantize.argtypes = [c_p, ctypes.c_int, i64, i64, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_double, c_p, c_p, c_p, c_p, c_p, ctypes.c_int]
        L.fo_quantize.restype = ctypes.c_int
        L.fo_quantize_2d.argtypes = [c_p, ctypes.c_int, i64, i64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, c_p, c_p, c_p, ctypes.c_int]
        L.fo_quantize_2d.restype = ctypes.c_int
        L.fo_dequantize.argtypes = [c_p, c_p, i64, i64, ctypes.c_double, c_p, ctypes.c_int]
        L.fo_dequantize.restype = ctypes.c_int
        L.fo_amax.argtypes = [c_p, ctypes.c_int, i64, ctypes.POINTER(ctypes.c_double)]
        L.fo_amax.restype = ctypes.c_int
        L.fo_tensor_scale.argtypes = [ctypes.c_double] * 3
        L.fo_tensor_scale.restype = ctypes.c_double
        L.fo_encode_fp4_rne.argtypes = [ctypes.c_double]
        L.fo_encode_fp4_rne.restype = ctypes.c_uint8
        L.fo_encode_e4m3.argtypes = [ctypes.c_double]
        L.fo_encode_e4m3.restype = ctypes.c_uint8
        L.fo_decode_e4m3.argtypes = [ctypes.c_uint8]
        L.fo_decode_e4m3.restype = ctypes.c_double
        L.fo_decode_fp4.argtypes = [ctypes.c_uint8]
        L.fo_decode_fp4.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def as_oracle_input(x: np.ndarray):
    """Return (contiguous array, dtype code).  bf16 is passed as uint16 bits."""
    x = np.ascontiguousarray(x)
    if x.dtype == np.float32:
        return x, DT_F32
    if x.dtype == np.uint16:
        return x, DT_BF16
    return np.ascontiguousarray(x, dtype=np.float64), DT_F64


def amax(x: np.ndarray, dtype_code: int | None = None):
    if dtype_code is None:
        x, dtype_code = as_oracle_input(x)
    out = ctypes.c_double()
    rc = lib().fo_amax(_ptr(x), dtype_code, x.size, ctypes.byref(out))
    return out.value, rc == 0


def tensor_scale(amax_v: float, m_fp4: float, fp8_cap: float) -> float:
    """blockquant.py:215-222 (alpha rounded through float32)."""
    return lib().fo_tensor_scale(amax_v, m_fp4, fp8_cap)


def m_tensor_cap(mode: str, fp8_cap: float | None = None):
    """QuantConfig.m_tensor / fp8_cap (blockquant.py:111-133)."""
    if mode == "adaptive":
        return 6.0, 256.0
    cap = 448.0 if fp8_cap is None else float(fp8_cap)
    return (4.0 if mode == "fixed4" else 6.0), cap


def quantize(x: np.ndarray, mode: str = "adaptive", rule: str = "mse", alpha=None,
             fp8_cap=None, want_errors: bool = False, nthreads: int = 0):
    """1-D 16-blocked quantization of x viewed as [rows, last].

    Returns dict(alpha, codes [rows, nb*8] packed, scales [rows, nb],
    pick4 [rows, nb], (err6, err4)).  x may be float32, float64 or uint16
    (bf16 bit patterns).
    """
    shape = x.shape
    x, dt = as_oracle_input(x)
    if x.ndim == 0 or x.size == 0:
        raise ValueError("oracle: tensor must be non-empty with ndim >= 1")
    cols = shape[-1]
    rows = x.size // cols
    if alpha is None:
        a, finite = amax(x, dt)
        if not finite:
            raise ValueError("oracle: non-finite input")
        alpha = tensor_scale(a, *m_tensor_cap(mode, fp8_cap))
    nb = (cols + 15) // 16
    codes = np.zeros((rows, nb * 8), np.uint8)
    scales = np.zeros((rows, nb), np.uint8)
    pick4 = np.zeros((rows, nb), np.uint8)
    e6 = np.zeros((rows, nb), np.float64) if want_errors else None
    e4 = np.zeros((rows, nb), np.float64) if want_errors else None
    rc = lib().fo_quantize(_ptr(x), dt, rows, cols, MODES[mode], RULES[rule], float(alpha),
                           _ptr(codes), _ptr(scales), _ptr(pick4), _ptr(e6), _ptr(e4),
                           int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle quantize failed rc={rc}")
    out = dict(alpha=float(alpha), codes=codes, scales=scales, pick4=pick4)
    if want_errors:
        out["err6"], out["err4"] = e6, e4
    return out


def quantize_2d(W: np.ndarray, mode: str = "adaptive", rule: str = "mse", alpha=None,
                fp8_cap=None, nthreads: int = 0):
    """16x16-tile weight quantization (transforms.py:134-179)."""
    W, dt = as_oracle_input(W)
    R, C = W.shape
    if alpha is None:
        a, finite = amax(W, dt)
        if not finite:
            raise ValueError("oracle: non-finite input")
        alpha = tensor_scale(a, *m_tensor_cap(mode, fp8_cap))
    nb = (C + 15) // 16
    codes = np.zeros((R, nb * 8), np.uint8)
    scales = np.zeros((R, nb), np.uint8)
    pick4 = np.zeros((R, nb), np.uint8)
    lib().fo_quantize_2d(_ptr(W), dt, R, C, MODES[mode], RULES[rule], float(alpha),
                         _ptr(codes), _ptr(scales), _ptr(pick4), int(nthreads))
    return dict(alpha=float(alpha), codes=codes, scales=scales, pick4=pick4)


def dequantize(codes: np.ndarray, scales: np.ndarray, alpha: float, rows: int, cols: int,
               nthreads: int = 0) -> np.ndarray:
    """blockquant.py:363-376; exact float64 result."""
    codes = np.ascontiguousarray(codes, np.uint8)
    scales = np.ascontiguousarray(scales, np.uint8)
    out = np.empty((rows, cols), np.float64)
    rc = lib().fo_dequantize(_ptr(codes), _ptr(scales), rows, cols, float(alpha), _ptr(out),
                             int(nthreads))
    if rc != 0:
        raise ValueError("oracle: NaN scale code")
    return out


def unpack_codes(packed: np.ndarray, cols: int) -> np.ndarray:
    """[rows, nb*8] packed -> [rows, cols] one code per element (reference layout)."""
    lo = packed & 0x0F
    hi = packed >> 4
    out = np.empty((packed.shape[0], packed.shape[1] * 2), np.uint8)
    out[:, 0::2] = lo
    out[:, 1::2] = hi
    return out[:, :cols]


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """[rows, cols] unpacked -> [rows, nb*8] packed with zero tail pads."""
    rows, cols = codes.shape
    nb = (cols + 15) // 16
    pad = np.zeros((rows, nb * 16), np.uint8)
    pad[:, :cols] = codes
    return (pad[:, 0::2] | (pad[:, 1::2] << 4)).astype(np.uint8)


def bf16_bits(x_f32: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (RNE) and return the uint16 bit patterns."""
    b = np.ascontiguousarray(x_f32, np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def apply_rht(x: np.ndarray, signs: np.ndarray) -> np.ndarray:
    """transforms.py:76-97 apply_rht restated: per contiguous group of 16
    along the last axis, y = fwht(g * signs) / sqrt(16) in float64, with the
    reference's butterfly order (h = 1, 2, 4, 8; top = a[j] + a[j+h],
    bot = a[j] - a[j+h] within each 2h-block).  Every output is the same single
    IEEE operation on the same operands as the reference's, so it is bit-exact."""
    a = np.asarray(x, dtype=np.float64)
    n = a.shape[-1]
    if n % 16:
        raise ValueError("oracle: last dimension must be a multiple of 16")
    g = a.reshape(-1, 16) * np.asarray(signs, dtype=np.float64)
    h = 1
    while h < 16:
        g = g.reshape(-1, 16 // (2 * h), 2, h)
        top = g[:, :, 0, :] + g[:, :, 1, :]
        bot = g[:, :, 0, :] - g[:, :, 1, :]
        g = np.stack([top, bot], axis=2).reshape(-1, 16)
        h *= 2
    return (g / np.sqrt(16.0)).reshape(a.shape)
