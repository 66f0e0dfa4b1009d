"""Row-sharded 4/6 quantization across ranks (one process per GPU).

The reference quantizes one tensor in one process (blockquant.py:334-360,
adaptive.py:83-101).  Its only cross-block dependency is the tensor scale
alpha = f32(max|X|) / f32(M * cap) (blockquant.py:215-222): given alpha, every
16-element block is independent.  Sharding a tensor by
contiguous row slabs therefore needs exactly one exchange -- an all-reduce
(MAX) of the per-shard amax -- after which each rank quantizes its slab with
the global alpha; the concatenated shards are bit-identical to the unsharded
call.

Slabs are multiples of 128 rows so no 128x4 tcgen05 scale tile straddles two
ranks.

Two layers:

* ``quantize_row_sharded`` is the protocol with the per-shard kernels passed
  in, so the same three steps run on B200s and, in the CPU tests, on the
  oracle over gloo (tests/test_sharded.py).
* ``ShardedQuantizer`` is the B200 product path: K1 (``f46_amax``) -> one
  in-place NCCL ``all_reduce(MAX)`` of the 8-byte float64 amax -> K2
  (``f46_quantize``) into preallocated per-rank buffers, all stream-ordered on
  the current stream (bench.py's timed step; tests/test_gpu_headline.py checks
  it against the oracle with the bench's own tensors).
"""

from __future__ import annotations

from typing import Callable, Optional

__all__ = ["shard_rows", "global_amax", "quantize_row_sharded", "ShardedQuantizer",
           "nccl_max_allreduce"]

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
    ``nccl_max_allreduce()``); with none the call is the single-process
    identity.  max is exact and order-independent, so every rank ends with the
    same bits.
    """
    if all_reduce_max is not None:
        all_reduce_max(local_amax)
    return local_amax


def quantize_row_sharded(x_local, amax_fn: Callable, quantize_fn: Callable,
                         all_reduce_max: Optional[Callable] = None):
    """amax (local) -> all-reduce MAX -> quantize the local slab with the global amax.

    amax_fn(x_local) -> 1-element amax tensor; quantize_fn(x_local, amax) ->
    quantized shard.
    """
    amax = amax_fn(x_local)
    amax = global_amax(amax, all_reduce_max)
    return quantize_fn(x_local, amax)


def nccl_max_allreduce(group=None) -> Optional[Callable]:
    """In-place MAX all-reduce over `group` with torch.distributed, or None
    when the job has a single rank (no collective is issued at all)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return None

    def reduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)

    return reduce


class ShardedQuantizer:
    """Quantize this rank's row slab of a row-sharded tensor with the global
    alpha.

    Buffers are allocated once for a fixed slab shape, so the per-step work is
    exactly two kernel launches and, for world > 1, one 8-byte NCCL
    all-reduce -- no allocation, no host synchronisation.
    """

    def __init__(self, rows: int, cols: int, dtype, device, mode: str = "adaptive",
                 fp8_cap: float = 256.0, all_reduce_max: Optional[Callable] = None):
        import torch

        from . import _lib
        from .blockquant import _DT_OF, scales_tc_bytes

        if mode not in _lib.MODE:
            raise ValueError(f"unknown mode {mode!r}")
        if mode == "adaptive" and fp8_cap != 256.0:
            raise ValueError("adaptive mode requires fp8_cap == 256")
        self.rows, self.cols, self.mode = int(rows), int(cols), mode
        self.dt = _DT_OF[dtype]
        self.mcap = (4.0 if mode == "fixed4" else 6.0) * float(fp8_cap)
        nb = -(-self.cols // 16)
        self.codes = torch.empty((self.rows, nb * 8), dtype=torch.uint8, device=device)
        self.scales_tc = torch.zeros(scales_tc_bytes(self.rows, self.cols), dtype=torch.uint8,
                                     device=device)
        # [amax (float64), barrier counter] for f46_quantize_fused; amax is its first word
        self.work = torch.zeros(2, dtype=torch.float64, device=device)
        self.amax = self.work[:1]
        self.alpha = torch.empty(1, dtype=torch.float64, device=device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=device)
        self.all_reduce_max = all_reduce_max
        self._L = _lib.load()
        self._lib = _lib
        from .blockquant import FUSED_MAX_BYTES

        esz = torch.empty(0, dtype=dtype).element_size()
        self.fused = self.rows * self.cols * esz <= FUSED_MAX_BYTES

    def amax_local(self, x, stream: int) -> None:
        """K1 over the local slab into self.amax (zeroed first)."""
        self.amax.zero_()
        self._lib.check(self._L.f46_amax(x.data_ptr(), self.dt, x.numel(), self.amax.data_ptr(),
                                         stream), "f46_amax")

    def exchange(self) -> None:
        """The one collective: in-place MAX all-reduce of the float64 amax."""
        global_amax(self.amax, self.all_reduce_max)

    def quantize_local(self, x, stream: int, flags: bool = False) -> None:
        """K2 over the local slab with alpha from the (global) amax."""
        L = self._L
        self._lib.check(L.f46_quantize(
            x.data_ptr(), self.dt, self.rows, self.cols, self._lib.MODE[self.mode], 0, self.mcap,
            self.amax.data_ptr(), 0.0, self.codes.data_ptr(), self.scales_tc.data_ptr(), None,
            None, self.alpha.data_ptr(), self.flags.data_ptr() if flags else None, stream),
            "f46_quantize")

    def __call__(self, x, stream: Optional[int] = None) -> None:
        import torch

        if tuple(x.shape) != (self.rows, self.cols) or not x.is_contiguous():
            raise ValueError(f"expected a contiguous ({self.rows}, {self.cols}) slab")
        s = torch.cuda.current_stream().cuda_stream if stream is None else stream
        if self.all_reduce_max is None and self.fused:
            # single rank, L2-sized slab: one cooperative launch (f46_quantize_fused)
            self.work.zero_()
            rc = self._L.f46_quantize_fused(
                x.data_ptr(), self.dt, self.rows, self.cols, self._lib.MODE[self.mode], 0, self.mcap,
                self.work.data_ptr(), self.codes.data_ptr(), self.scales_tc.data_ptr(),
                self.alpha.data_ptr(), None, s)
            if rc == self._lib.F46_OK:
                return
            self.fused = False
        self.amax_local(x, s)
        self.exchange()
        self.quantize_local(x, s)

    def container(self, shape=None):
        """The slab's result as a QuantizedTensor (views of the buffers)."""
        from .blockquant import QuantizedTensor

        return QuantizedTensor._from_device(shape or (self.rows, self.cols), "nvfp4", self.codes,
                                            self.scales_tc, self.alpha)
