"""Helpers to read the committed golden fixtures (tests/golden/*.npz,
generated from the real reference by tests/golden/make_golden.py)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    g = np.load(os.path.join(GOLDEN, name))
    out = []
    for n in g["__names__"]:
        n = str(n)
        rec = {k.split("::", 1)[1]: g[k] for k in g.files if k.startswith(n + "::")}
        out.append((n, rec))
    return out


def quant_cases():
    return load("golden_quant.npz")


def opt(v):
    v = float(v)
    return None if np.isnan(v) else v
