"""Multi-rank row-sharded quantization on CPU (gloo, world_size 2 and 4).

Each rank quantizes its row slab with the CPU oracle after an all-reduce(MAX)
of the per-shard amax over gloo (paper_2512_02010_b200.sharded); rank 0
gathers the shards and checks they are bit-identical to the unsharded oracle
call -- the property the NCCL path on B200s relies on.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_02010_b200.sharded import quantize_row_sharded, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tensor(rows, cols, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(rows, cols, generator=g).to(torch.bfloat16)
    return x.view(torch.int16).numpy().view(np.uint16)


def _worker(rank, world, port, rows, cols, seed, mode, out_dir):
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bits = _tensor(rows, cols, seed)
        r0, r1 = shard_rows(rows, world, rank)
        local = bits[r0:r1]
        mcap = O.m_tensor_cap(mode)

        def amax_fn(x):
            a, ok = O.amax(x) if x.size else (0.0, True)
            assert ok
            return torch.tensor([a], dtype=torch.float64)

        def quantize_fn(x, amax):
            alpha = O.tensor_scale(float(amax.item()), *mcap)
            return O.quantize(x, mode, alpha=alpha) if x.size else None

        q = quantize_row_sharded(local, amax_fn, quantize_fn,
                                 lambda t: dist.all_reduce(t, op=dist.ReduceOp.MAX))
        np.savez(os.path.join(out_dir, f"shard{rank}.npz"), codes=q["codes"], scales=q["scales"],
                 pick4=q["pick4"], alpha=q["alpha"])
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["adaptive", "fixed6"])
def test_row_sharded_equals_unsharded(tmp_path, world, mode):
    from oracle import oracle as O

    rows, cols, seed = 512 + 64, 256, 2  # last slab partial
    mp.spawn(_worker, args=(world, _free_port(), rows, cols, seed, mode, str(tmp_path)),
             nprocs=world, join=True)
    ref = O.quantize(_tensor(rows, cols, seed), mode)
    parts = [np.load(tmp_path / f"shard{r}.npz") for r in range(world)]
    assert all(float(p["alpha"]) == ref["alpha"] for p in parts)
    assert np.array_equal(np.concatenate([p["codes"] for p in parts]), ref["codes"])
    assert np.array_equal(np.concatenate([p["scales"] for p in parts]), ref["scales"])
    assert np.array_equal(np.concatenate([p["pick4"] for p in parts]), ref["pick4"])


def test_shard_rows_partition():
    for rows in (1, 127, 128, 129, 65536, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(rows, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and (a0 % 128 == 0 or a0 == rows)
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) < 256  # one 128-row unit + the partial tail
