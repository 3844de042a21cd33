"""The committed golden vectors (tests/golden/field_vectors.npz) against the
oracle that wrote them (regression guard for tools/dump_golden.py) and
against the product library's host-side level table (grid.hpp:66-84)."""
import importlib.util
import os

import numpy as np
import pytest

import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dumper():
    spec = importlib.util.spec_from_file_location("dump_golden", os.path.join(ROOT, "tools", "dump_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("case", G.CASES)
def test_oracle_reproduces_golden(case):
    d = _dumper()
    fresh = {k.split("/", 1)[1]: v for k, v in d.case_vectors(case, d.CASES[case]).items()}
    gold = G.load(case)
    assert set(fresh) == set(gold)
    exact = ("grid", "mlp", "resolution", "row_offset", "params0_sha256", "params0_head", "mlp_params0", "X",
             "target", "rows", "weights", "grad_table_index", "params1_untouched_sha256")
    for k in exact:
        assert np.array_equal(fresh[k], gold[k]), k
    for k in set(gold) - set(exact):
        np.testing.assert_allclose(fresh[k], gold[k], rtol=1e-5, atol=1e-9, err_msg=k)


@pytest.mark.parametrize("case", G.CASES)
def test_golden_internal_consistency(case):
    v = G.load(case)
    L, F = int(v["grid"][1]), int(v["grid"][3])
    B = v["X"].shape[0]
    nc = 1 << int(v["grid"][0])
    assert v["rows"].shape == (L, B, nc) and v["Y"].shape == (B, L * F)
    # the per-sample corner weights form a partition of unity (grid.hpp:180-212)
    assert np.allclose(v["weights"].sum(axis=2), 1.0, atol=1e-5)
    # touched table entries lie on the gathered rows
    rows = (v["row_offset"][:, None, None] + v["rows"].astype(np.int64)).ravel()
    ent = np.unique((rows[:, None] * F + np.arange(F)).ravel())
    assert np.isin(v["grad_table_index"], ent).all()
    # Adam moved every touched entry (lr 1e-2 >> fp32 ulp of 1e-4-size tables)
    assert (v["params1_table_touched"] != 0).all()


@pytest.mark.parametrize("case", G.CASES)
def test_library_level_table_matches_golden(case):   # grid.hpp:66-84 (host side of the C ABI)
    from paper_2201_05989_b200 import nf
    v = G.load(case)
    specs = nf.level_resolutions(nf.HashEncodingConfig(**G.grid_kwargs(v)))
    assert [s.resolution for s in specs] == v["resolution"].tolist()
    assert [s.row_offset for s in specs] == v["row_offset"].tolist()
