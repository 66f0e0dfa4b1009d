"""Row-sharded 4/6 quantization over NCCL with the CUDA kernels (world 2):
each rank quantizes its slab through sharded.ShardedQuantizer (K1 ->
all_reduce(MAX) -> K2); rank 0 gathers and checks the concatenation against
the oracle of the whole tensor.  Needs >= 2 GPUs; skipped otherwise."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import bench
    from paper_2512_02010_b200.blockquant import tc_to_rowmajor
    from paper_2512_02010_b200.sharded import ShardedQuantizer, nccl_max_allreduce

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        x = bench.c3_slab(dev, rank, world)[:2048].contiguous()
        sq = ShardedQuantizer(x.shape[0], x.shape[1], torch.bfloat16, dev, "adaptive",
                              all_reduce_max=nccl_max_allreduce())
        sq(x)
        torch.cuda.synchronize()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=x.cpu().view(torch.int16).numpy(),
                 codes=sq.codes.cpu().numpy(),
                 scales=tc_to_rowmajor(sq.scales_tc, x.shape[0], x.shape[1] // 16).cpu().numpy(),
                 alpha=sq.alpha.item())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_nccl_two_ranks(tmp_path):
    from oracle import oracle as O

    mp.spawn(_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    whole = np.concatenate([p["x"] for p in parts]).view(np.uint16)
    ref = O.quantize(whole, "adaptive")
    assert all(float(p["alpha"]) == ref["alpha"] for p in parts)
    assert np.array_equal(np.concatenate([p["codes"] for p in parts]), ref["codes"])
    assert np.array_equal(np.concatenate([p["scales"] for p in parts]), ref["scales"])
