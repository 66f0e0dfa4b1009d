"""Parity at the headline configurations' stated sizes, on the exact tensors
bench.py times (bench.c3_slab / c4_operands / moe_tensors / moe_step).

* C3 (65536 x 4096 BF16, BASELINE config 3): the timed K2 instantiation
  (``f46_quantize`` with no row-major scales and no pick4 output, called
  through sharded.ShardedQuantizer exactly as bench.py's step does) against the
  CPU oracle, bit for bit: packed codes, tcgen05 scales, alpha; the parity
  variant (row-major scales + pick4) against the oracle's 4/6 choice.
* C3 row-sharded on one GPU: the bench's per-rank slabs for world 2, 4, 8,
  per-slab K1 folded into one amax, each slab quantized with the global alpha;
  concatenated == the oracle of the whole tensor (SURVEY.md 8(e),
  reference blockquant.py:215-222).
* C4 8192^3: operands bit-exact vs the oracle, then the GEMM (f32 and bf16
  out) vs the float64 product of the exactly dequantized operands, relative
  Frobenius <= 1e-5 (the reference's bound, test_acceptance.py:191-198).
* C5: the bench's full MoE step (16 experts, all six expert GEMM shapes)
  against per-expert float64 products.
"""

import numpy as np
import pytest
import torch

import bench
import paper_2512_02010_b200 as f46
from oracle import oracle as O
from paper_2512_02010_b200.blockquant import tc_to_rowmajor
from paper_2512_02010_b200.sharded import ShardedQuantizer, shard_rows

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5


def bits_of(x: torch.Tensor) -> np.ndarray:
    return x.cpu().view(torch.int16).numpy().view(np.uint16)


def check_slab(sq, rows, ref, r0=0):
    r1 = r0 + rows
    got = sq.codes.cpu().numpy()
    bad = np.argwhere(got != ref["codes"][r0:r1])
    assert bad.size == 0, f"{len(bad)} code bytes differ, first at {bad[:4].tolist()}"
    sc = tc_to_rowmajor(sq.scales_tc, rows, bench.COLS // 16).cpu().numpy()
    assert np.array_equal(sc, ref["scales"][r0:r1])
    assert float(sq.alpha.item()) == ref["alpha"]


@pytest.fixture(scope="module")
def c3():
    dev = torch.device("cuda", 0)
    x = bench.c3_slab(dev, 0, 1)
    ref = O.quantize(bits_of(x), "adaptive")
    return x, ref


def test_c3_timed_instantiation_bit_exact(c3):
    x, ref = c3
    sq = ShardedQuantizer(x.shape[0], x.shape[1], torch.bfloat16, x.device, "adaptive")
    sq(x)
    torch.cuda.synchronize()
    check_slab(sq, x.shape[0], ref)


def test_c3_pick4_matches_oracle(c3):
    x, ref = c3
    q = f46.quantize_tensor_adaptive(x, f46.QuantConfig(scale_mode="adaptive"), want_pick4=True,
                                     want_rowmajor=True)
    assert np.array_equal(q.pick4.cpu().numpy(), ref["pick4"])
    assert np.array_equal(q.scales_rm.cpu().numpy(), ref["scales"])
    assert np.array_equal(q.packed_codes.cpu().numpy(), ref["codes"])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c3_row_sharded_on_one_gpu(world):
    """The bench's slabs for `world` ranks (seed 1234 + rank each): K1 per slab
    folded into one float64 amax (atomicMax is the MAX all-reduce's exact
    stand-in on one device), K2 per slab with the global alpha."""
    dev = torch.device("cuda", 0)
    slabs = [bench.c3_slab(dev, r, world) for r in range(world)]
    qs = [ShardedQuantizer(s.shape[0], s.shape[1], torch.bfloat16, dev, "adaptive") for s in slabs]
    amax = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    for s, q in zip(slabs, qs):
        q.amax_local(s, stream)
        torch.maximum(amax, q.amax, out=amax)
    for s, q in zip(slabs, qs):
        q.amax.copy_(amax)
        q.quantize_local(s, stream)
    whole = torch.cat(slabs)
    ref = O.quantize(bits_of(whole), "adaptive")
    r0 = 0
    for (a, b), q in zip([shard_rows(bench.ROWS, world, r) for r in range(world)], qs):
        assert a == r0
        check_slab(q, b - a, ref, r0)
        r0 = b
    assert r0 == bench.ROWS


def rel_fro(got, ref):
    return float(torch.linalg.norm(got.double() - ref) / torch.linalg.norm(ref))


def test_c4_8192_cubed():
    dev = torch.device("cuda", 0)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    xa, xb = bench.c4_operands(dev)
    aq = f46.quantize_tensor_adaptive(xa, cfg)
    bq = f46.quantize_tensor_adaptive(xb, cfg)
    for x, q in ((xa, aq), (xb, bq)):
        ref = O.quantize(bits_of(x), "adaptive")
        assert q.alpha == ref["alpha"]
        assert np.array_equal(q.packed_codes.cpu().numpy(), ref["codes"])
        assert np.array_equal(q.scale_codes, ref["scales"])
    # exact dequantization (f64) is itself pinned to the oracle (test_gpu_quant)
    a64 = f46.dequantize_tensor(aq, torch.float64)
    ra = O.quantize(bits_of(xa[:256]), "adaptive", alpha=aq.alpha)
    assert np.array_equal(a64[:256].cpu().numpy(),
                          O.dequantize(ra["codes"], ra["scales"], ra["alpha"], 256, 8192))
    ref = a64 @ f46.dequantize_tensor(bq, torch.float64).T
    del a64
    c32 = f46.gemm_nvfp4(aq, bq, torch.float32)
    assert rel_fro(c32, ref) <= REL_TOL
    c16 = f46.gemm_nvfp4(aq, bq, torch.bfloat16)
    assert torch.equal(c16.float(), f46.round_to_bf16(c32))  # bf16 out = RNE of the f32 result


def test_c5_moe_step_all_shapes():
    dev = torch.device("cuda", 0)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    t = bench.moe_tensors(dev)
    outs, plan = bench.moe_step(t, cfg, out_dtype=torch.float32)
    E = t["x"].shape[0]
    assert len(outs) == 6
    for name, (a, b, M, N, K) in plan.items():
        C = outs[name]
        assert C.shape == (E, M, N), name
        for e in range(E):
            ref = (f46.dequantize_tensor(a.group(e), torch.float64)
                   @ f46.dequantize_tensor(b.group(e), torch.float64).T)
            assert rel_fro(C[e], ref) <= REL_TOL, (name, e)


def test_c5_operands_match_oracle_one_expert():
    """The MoE step's quantized operands (one expert, every operand kind) are
    the oracle's containers bit for bit."""
    dev = torch.device("cuda", 0)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    t = bench.moe_tensors(dev, E=1)
    _, plan = bench.moe_step(t, cfg)
    x = t["x"][0]
    xq = plan["fprop_x_w1"][0].group(0)
    ref = O.quantize(bits_of(x), "adaptive")
    assert np.array_equal(xq.packed_codes.cpu().numpy(), ref["codes"])
    assert np.array_equal(xq.scale_codes, ref["scales"])
    w = t["W1"][0]
    wq = plan["fprop_x_w1"][1].group(0)
    r2 = O.quantize_2d(bits_of(w), "adaptive")
    assert wq.alpha == r2["alpha"]
    assert np.array_equal(wq.packed_codes.cpu().numpy(), r2["codes"])
    assert np.array_equal(wq.scale_codes, r2["scales"])
    # WGRAD operand: apply_rht(dy.T) along tokens, then 4/6 (qlinear.py:150-157)
    dy = t["dy"][0].cpu()
    spec = f46.RhtSpec(seed=cfg.seed)
    y = O.apply_rht(np.ascontiguousarray(dy.float().double().numpy().T), spec.signs)
    r3 = O.quantize(y, "adaptive")
    aq = plan["wgrad_dy_h"][0].group(0)
    assert aq.alpha == r3["alpha"]
    assert np.array_equal(aq.packed_codes.cpu().numpy(), r3["codes"])
    assert np.array_equal(aq.scale_codes, r3["scales"])
