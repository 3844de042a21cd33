"""Loader for tests/golden/field_vectors.npz (written by tools/dump_golden.py
from the pinned oracle)."""
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "field_vectors.npz")
CASES = ("small", "config1", "config2")


def load(case: str) -> dict:
    z = np.load(PATH)
    p = case + "/"
    return {k[len(p):]: z[k] for k in z.files if k.startswith(p)}


def grid_kwargs(v: dict) -> dict:
    d, L, T, F, nmin, nmax, smooth = (int(x) for x in v["grid"])
    return dict(dims=d, levels=L, table_size=T, features=F, n_min=nmin, n_max=nmax, interpolation=smooth)
