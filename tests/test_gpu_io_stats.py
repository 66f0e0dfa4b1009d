"""GPU: NVF4 container files and selection statistics vs the reference.

Files written from the device payload must be byte-identical to the ones the
reference's write_quantized produced for the same input (tensor_io.py:136-147,
fixtures from tests/golden/make_golden.py); reading a reference file yields
the same codes/scales/alpha.  The fused one-pass selection_stats matches the
reference's counts exactly and its aggregate MSE to 1e-12 (the reference's own
tolerance for this quantity, test_adaptive.py:199-205).
"""

import numpy as np
import pytest
import torch

import paper_2512_02010_b200 as f46
from oracle import oracle as O
from tests.golden_util import load

pytestmark = pytest.mark.gpu

CASES = load("golden_io.npz")


def to_torch(x):
    return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda()


def quant(rec):
    mode = str(rec["mode"])
    x = to_torch(rec["x"])
    if mode == "adaptive":
        return f46.quantize_tensor_adaptive(x, f46.QuantConfig(scale_mode="adaptive"))
    return f46.quantize_tensor(x, f46.QuantConfig(scale_mode=mode))


@pytest.mark.parametrize("name,rec", CASES, ids=[c[0] for c in CASES])
def test_written_file_is_byte_identical(tmp_path, name, rec):
    q = quant(rec)
    path = tmp_path / "q.nvf"
    f46.write_quantized(path, q)
    assert np.array_equal(np.frombuffer(path.read_bytes(), dtype=np.uint8), rec["file"])


@pytest.mark.parametrize("name,rec", CASES, ids=[c[0] for c in CASES])
def test_read_reference_file(tmp_path, name, rec):
    path = tmp_path / "ref.nvf"
    path.write_bytes(rec["file"].tobytes())
    r = f46.read_quantized(path)
    q = quant(rec)
    assert r == q
    assert torch.equal(f46.dequantize_tensor(r, torch.float64), f46.dequantize_tensor(q, torch.float64))


@pytest.mark.parametrize("name,rec", [c for c in CASES if "frac" in c[1]], ids=[c[0] for c in CASES if "frac" in c[1]])
def test_selection_stats_match_reference(name, rec):
    st = f46.selection_stats(to_torch(rec["x"]), f46.QuantConfig(scale_mode="adaptive"))
    assert st.n_blocks == int(rec["nblocks"])
    assert [st.fraction_4[r] for r in ("mse", "l1", "absmax")] == list(rec["frac"])
    assert [st.disagreements[k] for k in ("mse_vs_l1", "mse_vs_absmax", "l1_vs_absmax")] == list(rec["dis"])
    for got, want in zip([st.aggregate_mse[r] for r in ("mse", "l1", "absmax")], rec["agg"]):
        assert got == pytest.approx(float(want), rel=1e-12)


def test_selection_stats_large_matches_quantize_pick4():
    """mse-rule fraction equals the quantizer's own per-block choice (4096^2)."""
    g = torch.Generator().manual_seed(2)
    x = torch.randn(4096, 4096, generator=g).to(torch.bfloat16).cuda()
    cfg = f46.QuantConfig(scale_mode="adaptive")
    st = f46.selection_stats(x, cfg)
    q = f46.quantize_tensor_adaptive(x, cfg, want_pick4=True)
    assert st.fraction_4["mse"] == float(q.pick4.double().mean())
    mse = f46.reconstruction_mse(x, f46.dequantize_tensor(q, torch.float64))
    assert st.aggregate_mse["mse"] == pytest.approx(mse, rel=1e-12)


def test_selection_stats_fast_path_matches_float64_path():
    """BF16 input takes the f32-bracket codes, the same values as float64
    input the float64 restatement: identical counts and sums."""
    g = torch.Generator().manual_seed(23)
    x = torch.randn(1024, 2048, generator=g).to(torch.bfloat16)
    cfg = f46.QuantConfig(scale_mode="adaptive")
    a = f46.selection_stats(x.cuda(), cfg)
    b = f46.selection_stats(x.double().cuda(), cfg)
    assert a.fraction_4 == b.fraction_4
    assert a.disagreements == b.disagreements
    assert a.aggregate_mse == b.aggregate_mse


def test_selection_stats_rejects_nonfinite_with_alpha_override():
    x = torch.randn(32, 64).to(torch.bfloat16)
    x[3, 3] = float("nan")
    with pytest.raises(f46.InvalidInputError):
        f46.selection_stats(x.cuda(), f46.QuantConfig(scale_mode="adaptive"), alpha=0.01)


def test_reader_errors(tmp_path):
    p = tmp_path / "bad.nvf4"
    p.write_bytes(b"XXXX")
    with pytest.raises(f46.BadMagicError):
        f46.read_quantized(p)
    p.write_bytes(b"NVF4\x00")
    with pytest.raises(f46.TruncatedFileError):
        f46.read_quantized(p)
    p.write_bytes(b"NVF4\x07\x01" + (16).to_bytes(8, "little"))
    with pytest.raises(f46.UnsupportedDtypeError):
        f46.read_quantized(p)
    q = f46.quantize_tensor_adaptive(torch.randn(4, 16).cuda(), f46.QuantConfig(scale_mode="adaptive"))
    f46.write_quantized(p, q)
    p.write_bytes(p.read_bytes() + b"\x00")
    with pytest.raises(f46.FormatError):
        f46.read_quantized(p)
