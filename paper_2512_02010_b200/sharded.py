"""Row-sharded 4/6 quantization across ranks (one process per GPU).

The reference quantizes one tensor in one process (blockquant.py:334-360,
adaptive.py:83-101).  Its only cross-block dependency is the tensor scale
alpha = f32(max|X|) / f32(M * cap) (blockquant.py:215-222): given alpha, every
16-element block is independent.  Sharding a tensor by
contiguous row slabs therefore needs exactly one exchange -- an all-reduce
(MAX) of the per-shard amax -- after which each rank quantizes its slab with
the global alpha; the concatenated shards are bit-identical to the unsharded
call (tests/test_sharded.py checks this with the CPU oracle over gloo).

Slabs are multiples of 128 rows so no 128x4 tcgen05 scale tile straddles two
ranks.  The functions take the per-shard kernels as arguments so the same
protocol runs on B200s (libfouroversix, NCCL) and, in the CPU tests, on the
oracle (gloo).
"""

from __future__ import annotations

from typing import Callable, Optional

__all__ = ["shard_rows", "global_amax", "quantize_row_sharded"]

ROW_ALIGN = 128


def shard_rows(rows: int, world: int, rank: int, align: int = ROW_ALIGN) -> tuple[int, int]:
    """[begin, end) rows of `rank`: contiguous slabs, each a multiple of
    `align` rows except possibly the last, balanced to within one `align`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    units = -(-rows // align)
    per, rem = divmod(units, world)
    ub = rank * per + min(rank, rem)
    ue = ub + per + (1 if rank < rem else 0)
    return min(rows, ub * align), min(rows, ue * align)


def global_amax(local_amax, all_reduce_max: Optional[Callable] = None):
    """Fold the per-shard amax into the tensor-wide one (the single collective).

    `local_amax` is a 1-element tensor (float64 device tensor on B200s);
    `all_reduce_max` performs an in-place MAX all-reduce (for example
    ``lambda t: torch.distributed.all_reduce(t, op=ReduceOp.MAX)``); with
    none the call is the single-process identity.  max is exact and
    order-independent, so every rank ends with the same bits.
    """
    if all_reduce_max is not None:
        all_reduce_max(local_amax)
    return local_amax


def quantize_row_sharded(x_local, amax_fn: Callable, quantize_fn: Callable,
                         all_reduce_max: Optional[Callable] = None):
    """amax (local) -> all-reduce MAX -> quantize the local slab with the global amax.

    amax_fn(x_local) -> 1-element amax tensor; quantize_fn(x_local, amax) ->
    quantized shard.  On B200s these are blockquant.amax_device and
    quantize_1d(..., d_amax=amax); the kernels stay asynchronous on the
    current stream and the all-reduce is a 4..8-byte NCCL call.
    """
    amax = amax_fn(x_local)
    amax = global_amax(amax, all_reduce_max)
    return quantize_fn(x_local, amax)
