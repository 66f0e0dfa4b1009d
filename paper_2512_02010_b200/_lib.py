"""ctypes binding of libfouroversix.so, the C ABI declared in include/fouroversix.h.

The library is the only compute path of this package.  There is no CPU or
PyTorch fallback: if the shared object is missing, or no CUDA device is
present, every operation raises ``RuntimeError`` immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("F46_LIB_PATH") or os.path.join(_HERE, "libfouroversix.so")

# constants mirrored from include/fouroversix.h
F46_OK = 0
F46_ERR_INVALID_ARG = -1
F46_ERR_CONFIG = -2
F46_ERR_UNSUPPORTED = -3
F46_ERR_CUDA = -4

DT_F32, DT_BF16, DT_F64 = 0, 1, 2
FIXED6, FIXED4, ADAPTIVE = 0, 1, 2
RULE = {"mse": 0, "l1": 1, "absmax": 2}
MODE = {"fixed6": FIXED6, "fixed4": FIXED4, "adaptive": ADAPTIVE}
SCALES_TC, SCALES_RM = 0, 1
HOOK = {"seg_chunk_bytes": 0, "dq_vec": 1, "q2_v1": 2, "sr_one_thread": 3, "gemm_kernel": 4}
FLAG_NONFINITE = 1
FLAG_NAN_SCALE = 2

# every symbol include/fouroversix.h declares
EXPORTS = (
    "f46_scales_tc_bytes",
    "f46_codes_bytes",
    "f46_amax",
    "f46_quantize",
    "f46_quantize_2d",
    "f46_dequantize",
    "f46_gemm_nvfp4",
    "f46_gemm_nvfp4_grouped",
    "f46_gemm_nvfp4_amax",
    "f46_gemm_nvfp4_grouped_amax",
    "f46_selection_stats",
    "f46_quantize_sr",
    "f46_rht16",
    "f46_amax_grouped",
    "f46_quantize_grouped",
    "f46_quantize_2d_grouped",
    "f46_rht_t_amax_grouped",
    "f46_quantize_rht_t_grouped",
    "f46_quantize_block_ref",
    "f46_matmul_f32_ordered",
    "f46_set_test_hook",
    "f46_quantize_fused",
    "f46_build_info",
)

_lock = threading.Lock()
_lib = None


def _declare(L):
    p, i, i64, d, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
    L.f46_scales_tc_bytes.argtypes = [i64, i64]
    L.f46_scales_tc_bytes.restype = sz
    L.f46_codes_bytes.argtypes = [i64, i64]
    L.f46_codes_bytes.restype = sz
    L.f46_amax.argtypes = [p, i, i64, p, p]
    L.f46_amax.restype = i
    q_args = [p, i, i64, i64, i, i, d, p, d, p, p, p, p, p, p, p]
    L.f46_quantize.argtypes = q_args
    L.f46_quantize.restype = i
    L.f46_quantize_2d.argtypes = [p, i, i64, i64, i, i, d, p, d, p, p, p, p, p, p, p, p, p]
    L.f46_quantize_2d.restype = i
    L.f46_dequantize.argtypes = [p, p, i, p, i64, i64, p, i, p, p]
    L.f46_dequantize.restype = i
    L.f46_gemm_nvfp4.argtypes = [p, p, p, p, p, p, i64, i64, i64, p, i64, i, p]
    L.f46_gemm_nvfp4.restype = i
    L.f46_gemm_nvfp4_grouped.argtypes = [i, p, p, p, p, p, p, i64, i64, i64, p, i64, i, p]
    L.f46_gemm_nvfp4_grouped.restype = i
    L.f46_gemm_nvfp4_amax.argtypes = [p, p, p, p, p, p, i64, i64, i64, p, i64, i, p, p]
    L.f46_gemm_nvfp4_amax.restype = i
    L.f46_gemm_nvfp4_grouped_amax.argtypes = [i, p, p, p, p, p, p, i64, i64, i64, p, i64, i, p, p]
    L.f46_gemm_nvfp4_grouped_amax.restype = i
    L.f46_selection_stats.argtypes = [p, i, i64, i64, d, p, d, p, i, p, p]
    L.f46_selection_stats.restype = i
    u64 = ctypes.c_uint64
    L.f46_quantize_sr.argtypes = [p, i, i64, i64, i, i, d, p, d, u64, u64, u64, u64, p, p, p, p, p, p, p]
    L.f46_quantize_sr.restype = i
    L.f46_rht16.argtypes = [p, i, i64, p, p, p]
    L.f46_rht16.restype = i
    L.f46_amax_grouped.argtypes = [p, i, i, i64, p, p]
    L.f46_amax_grouped.restype = i
    L.f46_quantize_grouped.argtypes = [p, i, i, i64, i64, i, i, d, p, p, p, p, p, p]
    L.f46_quantize_grouped.restype = i
    L.f46_quantize_2d_grouped.argtypes = [p, i, i, i64, i64, i, i, d, p, p, p, p, p, p, p, p]
    L.f46_quantize_2d_grouped.restype = i
    u32 = ctypes.c_uint32
    L.f46_rht_t_amax_grouped.argtypes = [p, i, i, i64, i64, u32, p, p]
    L.f46_rht_t_amax_grouped.restype = i
    L.f46_quantize_rht_t_grouped.argtypes = [p, i, i, i64, i64, u32, i, i, d, p, p, p, p, p, p]
    L.f46_quantize_rht_t_grouped.restype = i
    L.f46_quantize_block_ref.argtypes = [p, i64, d, d, p, p, p, p, p]
    L.f46_quantize_block_ref.restype = i
    L.f46_matmul_f32_ordered.argtypes = [p, p, i64, i64, i64, p, p]
    L.f46_matmul_f32_ordered.restype = i
    L.f46_quantize_fused.argtypes = [p, i, i64, i64, i, i, d, p, p, p, p, p, p]
    L.f46_quantize_fused.restype = i
    L.f46_set_test_hook.argtypes = [i, i64]
    L.f46_set_test_hook.restype = i
    L.f46_build_info.argtypes = []
    L.f46_build_info.restype = ctypes.c_char_p


def load(require_symbols: bool = True):
    """Load (once) and return the ctypes handle; raise if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libfouroversix.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)"
                )
            L = ctypes.CDLL(LIB_PATH)
            _declare(L)
            _lib = L
    return _lib


def check(rc: int, what: str):
    """Map a C ABI return code onto the reference's exception convention."""
    if rc == F46_OK:
        return
    from .errors import ConfigError, InvalidInputError

    if rc == F46_ERR_INVALID_ARG:
        raise InvalidInputError(f"{what}: invalid argument")
    if rc == F46_ERR_CONFIG:
        raise ConfigError(f"{what}: invalid configuration")
    if rc == F46_ERR_UNSUPPORTED:
        raise InvalidInputError(f"{what}: unsupported shape or alignment")
    raise RuntimeError(f"{what}: CUDA launch failed (rc={rc})")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
