"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/nfg.h declares, and its host-only pieces (level table, hash,
lr_at) agree bit-for-bit with the oracle."""
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "nfg.h")).read()
    return sorted(set(re.findall(r"\b(nfg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_05989_b200 import _lib
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    from paper_2201_05989_b200 import _lib
    names = _declared()
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    assert lib.nfg_abi_version() == 4


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2201_05989_b200", "libnfg.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


@pytest.mark.parametrize("cfg", [
    dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048),
    dict(dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=1024),
    dict(dims=2, levels=16, table_size=1 << 24, features=2, n_min=16, n_max=8192),
    dict(dims=3, levels=8, table_size=1 << 12, features=4, n_min=2, n_max=300),
    dict(dims=2, levels=1, table_size=2, features=1, n_min=16, n_max=512),
])
def test_level_table_matches_oracle(cfg):   # grid.hpp:66-84, bit-exact
    from paper_2201_05989_b200 import nf
    a = nf.level_resolutions(nf.HashEncodingConfig(**cfg))
    b = O.level_resolutions(O.GridCfg(**cfg))
    assert [(x.resolution, x.table_len, x.dense, x.row_offset) for x in a] == \
        [(y.resolution, y.table_len, y.dense, y.row_offset) for y in b]


def test_invalid_config_rejected():   # grid.hpp:34-46
    from paper_2201_05989_b200 import nf
    from paper_2201_05989_b200._lib import NfgInvalidArgument
    for bad in (dict(levels=0), dict(table_size=100), dict(features=0), dict(n_min=0), dict(n_min=8, n_max=4),
                dict(dims=4)):
        with pytest.raises(NfgInvalidArgument):
            nf.level_resolutions(nf.HashEncodingConfig(**bad))


def test_hash_matches_oracle():   # grid.hpp:88-95
    from paper_2201_05989_b200 import nf
    rng = O.Pcg32(99, 1)
    for _ in range(500):
        c = [rng.next_u32(), rng.next_u32(), rng.next_u32()]
        for d in (1, 2, 3):
            for T in (16, 1 << 14, 1 << 19, 1 << 24):
                assert nf.spatial_hash(c, d, T) == O.spatial_hash(c, d, T)


def test_lr_at_and_default_schedule(kats):   # adam.hpp:139-161
    from paper_2201_05989_b200 import nf
    k = kats["lr_at"]
    s = nf.LrSchedule(k["milestones"], k["factor"])
    for step, lr in k["cases"]:
        assert nf.lr_at(s, k["base"], step) == O.lr_at(k["milestones"], k["factor"], k["base"], step)
    for total, ms in kats["default_schedule"]["cases"]:
        assert nf.default_schedule(total).milestones == ms


def test_context_fails_loudly_without_gpu():
    """No CPU fallback: without a usable GPU the context creation errors out."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2201_05989_b200 import nf
    from paper_2201_05989_b200._lib import NfgError
    with pytest.raises(NfgError):
        nf.Context(0)


def test_host_mirror_functions_match_oracle(kats):   # grid.hpp:100-110, losses.hpp:63-71
    import numpy as np
    import oracle as O
    from paper_2201_05989_b200 import nf
    cfg = nf.HashEncodingConfig(levels=6, table_size=1 << 10, features=2, n_min=4, n_max=64, dims=3)
    specs = nf.level_resolutions(cfg)
    ospecs = O.level_resolutions(O.GridCfg(levels=6, table_size=1 << 10, features=2, n_min=4, n_max=64, dims=3))
    rng = np.random.default_rng(1)
    for s, o in zip(specs, ospecs):
        for _ in range(50):
            c = rng.integers(0, s.resolution + 1, 3)
            assert nf.grid_vertex_index(s, c, 3, 1 << 10) == O.grid_vertex_index(o.resolution, o.dense, c, 3, 1 << 10)
    a = rng.uniform(size=(40, 3)).astype(np.float32)
    b = rng.uniform(size=(40, 3)).astype(np.float32)
    assert abs(nf.psnr(a, b) - O.psnr(a, b)) < 1e-9
    assert nf.psnr(a, a) == 100.0
