"""The oracle's RHT restatement (oracle.apply_rht, test infrastructure)
against the reference's own apply_rht outputs in the committed fixture
(tests/golden/make_golden.py sr_rht_cases) -- CPU only, bit for bit."""

import numpy as np

from oracle import oracle as O
from paper_2512_02010_b200.transforms import RhtSpec
from tests.golden_util import load


def test_rht_matches_reference_fixture():
    cases = [(n, r) for n, r in load("golden_sr.npz") if n.startswith("rht_")]
    assert cases
    for name, rec in cases:
        spec = RhtSpec(seed=int(rec["seed"]))
        assert np.array_equal(O.apply_rht(rec["x"], spec.signs), rec["y"]), name
