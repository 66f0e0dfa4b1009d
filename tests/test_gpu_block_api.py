"""The block-level API (any block length, any target m, RNE and stochastic
rounding with explicit uniforms) and emulated_fp4_matmul(transpose_b=False)
against outputs of the real reference (tests/golden/golden_block.npz, made by
tests/golden/make_golden.py block): codes, scale codes, the error means and
the dequantized block bit for bit; the NN matmul bit for bit (the reference's
ordered float32 accumulation)."""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from tests.golden_util import load

pytestmark = pytest.mark.gpu

CASES = load("golden_block.npz")
QB = [(n, r) for n, r in CASES if n.startswith(("qb_", "table2_"))]
QBA = [(n, r) for n, r in CASES if n.startswith("qba_")]
MM = [(n, r) for n, r in CASES if n.startswith("mm_nn_")]


@pytest.mark.parametrize("name,rec", QB, ids=[c[0] for c in QB])
def test_quantize_block_any_length_and_target(name, rec):
    rounding = str(rec["rounding"])
    r = f46.quantize_block(rec["x"], float(rec["alpha"]), float(rec["m"]), rounding=rounding,
                           u=rec["u"] if rounding == "sr" else None)
    assert np.array_equal(np.asarray(r.codes, np.uint8), rec["codes"])
    assert r.scale_code == int(rec["scale"])
    assert [r.err_mse, r.err_l1, r.err_max] == list(rec["err"])
    assert np.array_equal(np.asarray(r.dequant), rec["deq"])
    assert int(f46.compute_block_scale(rec["x"], float(rec["alpha"]), float(rec["m"]))) == int(rec["cbs"])


@pytest.mark.parametrize("name,rec", QBA, ids=[c[0] for c in QBA])
def test_quantize_block_adaptive_any_length(name, rec):
    rounding = str(rec["rounding"])
    sr = rounding == "sr"
    r = f46.quantize_block_adaptive(rec["x"], float(rec["alpha"]), rule=str(rec["rule"]),
                                    rounding=rounding, u6=rec["u6"] if sr else None,
                                    u4=rec["u4"] if sr else None)
    assert r.chosen_m == int(rec["m"])
    assert np.array_equal(np.asarray(r.codes, np.uint8), rec["codes"])
    assert r.scale_code == int(rec["scale"])
    assert [r.err_mse, r.err_l1, r.err_max] == list(rec["err"])


def bf16_tensor(bits):
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).cuda()


@pytest.mark.parametrize("name,rec", MM, ids=[c[0] for c in MM])
def test_emulated_matmul_nn_bit_exact(name, rec):
    cfg = f46.QuantConfig(scale_mode="adaptive")
    aq = f46.quantize_tensor_adaptive(bf16_tensor(rec["a"]), cfg)
    bq = f46.quantize_tensor_adaptive(bf16_tensor(rec["b"]), cfg)
    c = f46.emulated_fp4_matmul(aq, bq, transpose_b=False).cpu().numpy()
    assert np.array_equal(c, rec["c"])
    c16 = f46.emulated_fp4_matmul(aq, bq, transpose_b=False, bf16_out=True).cpu().numpy()
    assert np.array_equal(c16, rec["c16"])


def test_dequantize_default_is_the_exact_float64():
    x = (torch.randn(64, 64, generator=torch.Generator().manual_seed(3)) * 2).to(torch.bfloat16)
    q = f46.quantize_tensor_adaptive(x.cuda(), f46.QuantConfig(scale_mode="adaptive"))
    d = f46.dequantize_tensor(q)
    assert d.dtype == torch.float64
    assert torch.equal(d, f46.dequantize_tensor(q, torch.float64))
