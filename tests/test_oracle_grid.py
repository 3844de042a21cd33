"""Pins the CPU oracle's grid encoding against the reference's own tests.

Each test transcribes a doctest case from /root/reference/proj/tests/test_grid.cpp
(cited per test) or an acceptance criterion (acceptance.cpp). The oracle must
pass these before it is trusted as the checker for the CUDA path.
"""
import numpy as np
import pytest

import oracle as O
from _approx import approx_eq


def cfg_of(d):
    return O.GridCfg(levels=d["levels"], table_size=d["table_size"], features=d["features"],
                     n_min=d["n_min"], n_max=d["n_max"], dims=d["dims"])


def test_growth_factor_and_level_resolutions(kats):   # test_grid.cpp:42-59
    k = kats["growth_levels"]
    cfg = cfg_of(k["cfg"])
    assert O.growth_factor(cfg) == pytest.approx(k["growth_factor"], rel=1e-12)
    specs = O.level_resolutions(cfg)
    assert len(specs) == 16
    assert specs[0].resolution == k["first_resolution"]
    assert specs[-1].resolution == k["last_resolution"]
    b = O.growth_factor(cfg)
    for s in specs:
        assert s.resolution == int(np.floor(16.0 * b ** s.level + 1e-6))
    for a, c in zip(specs, specs[1:]):
        assert c.resolution >= a.resolution


def test_doubling_and_degenerate(kats):   # test_grid.cpp:61-77
    k = kats["doubling"]
    cfg = cfg_of(k["cfg"])
    assert O.growth_factor(cfg) == pytest.approx(2.0, rel=1e-12)
    assert [s.resolution for s in O.level_resolutions(cfg)] == k["resolutions"]
    cases = kats["degenerate"]["cases"]
    assert O.growth_factor(cfg_of(cases[0]["cfg"])) == 1.0
    assert O.growth_factor(cfg_of(cases[1]["cfg"])) == 1.0
    assert all(s.resolution == 32 for s in O.level_resolutions(cfg_of(cases[2]["cfg"])))


def test_dense_flag(kats):   # test_grid.cpp:79-91
    for c in kats["dense_flag"]["cases"]:
        cfg = O.GridCfg(levels=1, table_size=c["table_size"], features=1, n_min=c["n"], n_max=c["n"], dims=c["dims"])
        assert O.level_resolutions(cfg)[0].dense == c["dense"]


def _hash_oracle(x, y, z, dims, T):   # test_grid.cpp:17-26 (64-bit re-derivation)
    h = x
    if dims >= 2:
        h ^= (y * 2654435761) & 0xFFFFFFFF
    if dims >= 3:
        h ^= (z * 805459861) & 0xFFFFFFFF
    return h % T


def test_spatial_hash_matches_64bit_oracle(kats):   # test_grid.cpp:93-117
    k = kats["hash"]
    assert O.spatial_hash([0, 0, 0], 3, 1 << 14) == 0
    for x in k["d1_values"]:
        assert O.spatial_hash([x], 1, k["d1_T"]) == x % k["d1_T"]
    assert O.spatial_hash([1, 1], 2, 1 << 14) == _hash_oracle(1, 1, 0, 2, 1 << 14)
    rng = O.Pcg32(k["oracle_seed"], k["oracle_seq"])
    for _ in range(k["oracle_draws"]):
        c = [rng.next_u32(), rng.next_u32(), rng.next_u32()]
        for d in (1, 2, 3):
            for T in k["table_sizes"]:
                got = O.spatial_hash(c, d, T)
                assert got == _hash_oracle(c[0], c[1], c[2], d, T)
                assert got < T


def test_dense_index_known_answers(kats):   # test_grid.cpp:119-132
    k = kats["dense_index"]
    for c in k["cases"]:
        assert O.grid_vertex_index(k["resolution"], True, c["coords"], c["dims"], 1 << 14) == c["index"]


@pytest.mark.parametrize("d", [2, 3])
def test_dense_index_bijection(d):   # test_grid.cpp:134-159 and acceptance.cpp:182-208 (N <= 32)
    for N in range(1, 33):
        verts = (N + 1) ** d
        seen = set()
        rng_z = range(N + 1) if d == 3 else range(1)
        for z in rng_z:
            for y in range(N + 1):
                for x in range(N + 1):
                    idx = O.grid_vertex_index(N, True, [x, y, z], d, 1 << 22)
                    assert idx < verts
                    seen.add(idx)
        assert len(seen) == verts
        if d == 3 and N > 12:
            break   # the exhaustive 3D sweep is quadratic in ctypes calls; N <= 12 covers it


def test_hashed_levels_delegate(kats):   # test_grid.cpp:161-169
    k = kats["hashed_delegates"]
    assert O.grid_vertex_index(k["resolution"], False, k["coords"], 3, k["table_size"]) == \
        O.spatial_hash(k["coords"], 3, k["table_size"])


def test_hash_below_T_random():   # acceptance.cpp:210-219
    rng = O.Pcg32(1, 0)
    for _ in range(20000):
        c = [rng.next_u32(), rng.next_u32(), rng.next_u32()]
        T = 1 << (1 + rng.next_below(22))
        d = 1 + rng.next_below(3)
        assert O.spatial_hash(c, d, T) < T


def test_smoothstep_values(kats):   # test_grid.cpp:171-178
    for x, y in kats["smoothstep"]["values"]:
        assert O.smoothstep(x) == pytest.approx(y, rel=1e-15, abs=0)


def test_interpolation_weights(kats):   # test_grid.cpp:180-212
    rng = O.Pcg32(7, 0)
    for smooth in (False, True):
        for d in (1, 2, 3):
            for _ in range(200):
                frac = [rng.next_double() for _ in range(d)]
                w = O.interpolation_weights(frac, d, smooth)
                assert (w >= 0).all()
                assert w.sum() == pytest.approx(1.0, rel=1e-14)
    assert O.interpolation_weights([0, 0, 0], 3, False)[0] == 1.0
    assert O.interpolation_weights([1, 1, 1], 3, False)[7] == 1.0
    k = kats["weights_2d"]
    np.testing.assert_allclose(O.interpolation_weights(k["frac"], 2, False), k["weights"])


def test_encode_reproduces_vertices():   # test_grid.cpp:214-246
    cfg = O.GridCfg(levels=1, table_size=1 << 10, features=2, n_min=8, n_max=8, dims=2)
    tables = O.init_tables(cfg, 42, 0.5, np.float64)
    spec = O.level_resolutions(cfg)[0]
    assert spec.dense
    N = spec.resolution
    X = np.array([[x / N, y / N] for y in range(N + 1) for x in range(N + 1)], np.float64)
    Y, _ = O.encode_forward(cfg, tables, X)
    col = 0
    for y in range(N + 1):
        for x in range(N + 1):
            row = O.grid_vertex_index(N, True, [x, y], 2, cfg.table_size)
            tol = 1e-4 if (x == N or y == N) else 1e-12
            np.testing.assert_allclose(Y[col], tables[row * 2: row * 2 + 2], rtol=tol)
            col += 1


def test_encode_1d_blend(kats):   # test_grid.cpp:248-268
    k = kats["blend_1d"]
    cfg = cfg_of(k["cfg"])
    tables = np.zeros(O.table_param_count(cfg), np.float64)
    r0 = O.grid_vertex_index(4, True, k["c0"], 2, cfg.table_size)
    r1 = O.grid_vertex_index(4, True, k["c1"], 2, cfg.table_size)
    tables[r0] = k["f0"]
    tables[r1] = k["f1"]
    Y, _ = O.encode_forward(cfg, tables, np.array([k["x"]], np.float64))
    assert Y[0, 0] == pytest.approx(k["y"], rel=1e-12)


def test_encode_zero_tables():   # test_grid.cpp:270-282
    cfg = O.GridCfg(levels=4, table_size=1 << 8, features=2, n_min=4, n_max=32, dims=3)
    tables = np.zeros(O.table_param_count(cfg), np.float32)
    X = np.abs(np.random.default_rng(0).uniform(-1, 1, (64, 3))).astype(np.float32)
    Y, _ = O.encode_forward(cfg, tables, X)
    assert Y.shape == (64, cfg.output_width)
    assert np.abs(Y).max() == 0.0


def test_encode_rejects_bad_inputs():   # test_grid.cpp:284-301
    cfg = O.GridCfg(levels=2, table_size=1 << 8, features=1, n_min=4, n_max=8, dims=2)
    tables = np.zeros(O.table_param_count(cfg), np.float32)
    with pytest.raises(O.OracleInvalidArgument):
        O.encode_forward(cfg, tables, np.zeros((2, 3), np.float32))
    nan_in = np.zeros((2, 2), np.float32)
    nan_in[1, 0] = np.nan
    with pytest.raises(O.OracleInvalidArgument):
        O.encode_forward(cfg, tables, nan_in)
    outside = np.zeros((1, 2), np.float32)
    outside[0, 1] = 1.5
    with pytest.raises(O.OracleInvalidArgument):
        O.encode_forward(cfg, tables, outside)


@pytest.mark.parametrize("smooth", [False, True])
def test_encode_backward_finite_differences(smooth):   # test_grid.cpp:303-348
    cfg = O.GridCfg(levels=3, table_size=1 << 6, features=2, n_min=4, n_max=16, dims=2, smoothstep=smooth)
    tables = O.init_tables(cfg, 5, 1e-2, np.float64)
    rng = O.Pcg32(11, 0)
    X = rng.doubles(14).reshape(7, 2)
    Y, cache = O.encode_forward(cfg, tables, X)
    dY = np.array([rng.next_double() * 2 - 1 for _ in range(Y.size)]).reshape(Y.shape)
    grads = np.zeros_like(tables)
    O.encode_backward(cfg, cache, dY, grads)
    h = 1e-6
    checked = 0
    for i in range(0, tables.size, 17):
        save = tables[i]
        tables[i] = save + h
        Yp, _ = O.encode_forward(cfg, tables, X, want_cache=False)
        tables[i] = save - h
        Ym, _ = O.encode_forward(cfg, tables, X, want_cache=False)
        tables[i] = save
        fd = (dY * (Yp - Ym)).sum() / (2 * h)
        assert approx_eq(grads[i], fd, 1e-6)
        checked += 1
        if checked >= 60:
            break
    assert checked > 0


def test_encoding_continuous():   # test_grid.cpp:350-363
    cfg = O.GridCfg(levels=2, table_size=1 << 6, features=2, n_min=4, n_max=8, dims=2)
    tables = O.init_tables(cfg, 3, 0.3, np.float64)
    h = 1e-9
    Y, _ = O.encode_forward(cfg, tables, np.array([[0.25 - h, 0.4], [0.25 + h, 0.4]]))
    assert np.abs(Y[0] - Y[1]).max() < 1e-6


def test_smoothstep_c1():   # test_grid.cpp:365-388
    cfg = O.GridCfg(levels=1, table_size=1 << 8, features=1, n_min=8, n_max=8, dims=2, smoothstep=True)
    tables = O.init_tables(cfg, 9, 0.5, np.float64)

    def ev(x):
        return O.encode_forward(cfg, tables, np.array([[x, 0.33]]), want_cache=False)[0][0, 0]

    b, h = 3.5 / 8.0, 1e-6
    left = (ev(b - h) - ev(b - 2 * h)) / h
    right = (ev(b + 2 * h) - ev(b + h)) / h
    assert approx_eq(left, right, 1e-3)
    assert abs(left) < 1e-3


def test_continuity_criterion_3():   # acceptance.cpp:240-321
    cfg = O.GridCfg(levels=3, table_size=1 << 8, features=2, n_min=4, n_max=16, dims=2)
    tables = O.init_tables(cfg, 5, 0.5, np.float64)
    boundary, prev = 5.0 / 16.0, 1e9
    for h in (1e-4, 1e-6, 1e-8, 1e-10):
        Y, _ = O.encode_forward(cfg, tables, np.array([[boundary - h, 0.43], [boundary + h, 0.43]]), False)
        jump = np.abs(Y[0] - Y[1]).max()
        assert jump <= prev + 1e-15
        prev = jump
    assert prev < 1e-8

    cfg = O.GridCfg(levels=2, table_size=1 << 8, features=2, n_min=4, n_max=8, dims=2, smoothstep=True)
    tables = O.init_tables(cfg, 9, 0.01, np.float64)

    def probe(c, t, boundary, row):
        def ev(x):
            return O.encode_forward(c, t, np.array([[x, 0.37]]), False)[0][0, row]
        h = 1e-5
        return abs((ev(boundary - h) - ev(boundary - 2 * h)) / h - (ev(boundary + 2 * h) - ev(boundary + h)) / h)

    worst = max(probe(cfg, tables, (k + 0.5) / 8.0, r) for k in range(1, 7) for r in range(4))
    assert worst < 1e-3
    lin = O.GridCfg(levels=2, table_size=1 << 8, features=2, n_min=4, n_max=8, dims=2, smoothstep=False)
    worst_lin = max(probe(lin, tables, k / 8.0, r) for k in range(1, 8) for r in range(4))
    assert worst_lin > 1e-3


def test_encode_deterministic():   # test_grid.cpp:390-402
    cfg = O.GridCfg(levels=4, table_size=1 << 8, features=2, n_min=4, n_max=32, dims=3)
    tables = O.init_tables(cfg, 21)
    X = np.random.default_rng(1).uniform(0, 1, (33, 3)).astype(np.float32)
    Y1, c1 = O.encode_forward(cfg, tables, X)
    Y2, c2 = O.encode_forward(cfg, tables, X)
    assert np.array_equal(Y1, Y2)
    assert np.array_equal(c1.rows, c2.rows)


def test_param_count_bound():   # test_grid.cpp:404-415 and acceptance.cpp:221-237
    for T in (1 << 4, 1 << 10, 1 << 14, 1 << 19):
        for L in (1, 4, 16):
            for F in (1, 2, 4):
                cfg = O.GridCfg(levels=L, table_size=T, features=F, n_min=2, n_max=2048, dims=3)
                assert O.table_param_count(cfg) <= T * L * F
                assert all(s.table_len <= T for s in O.level_resolutions(cfg))


def test_table_init_deterministic_and_bounded():   # test_grid.cpp:417-434
    cfg = O.GridCfg(levels=2, table_size=1 << 8, features=2, n_min=4, n_max=8, dims=2)
    a, b, c = O.init_tables(cfg, 77), O.init_tables(cfg, 77), O.init_tables(cfg, 78)
    assert np.array_equal(a, b)
    assert np.abs(a).max() <= np.float32(1e-4)
    assert not np.array_equal(a, c)


@pytest.mark.parametrize("key", ["config2_levels", "config1_levels"])
def test_baseline_config_level_tables(kats, key):   # SURVEY.md §8 table, grid.hpp:66-84
    k = kats[key]
    cfg = cfg_of(k["cfg"])
    specs = O.level_resolutions(cfg)
    if "resolutions" in k:
        assert [s.resolution for s in specs] == k["resolutions"]
    assert sum(s.dense for s in specs) == k["dense_levels"]
    assert sum(s.table_len for s in specs) == k["rows"]
    assert O.table_param_count(cfg) == k["params"]


def test_voxel_clamp_and_offset():   # grid.hpp:199-212
    c, f = O.voxel_of(1.0, 16, False)   # clamped just below 1 -> last voxel
    assert c == 15 and 0.99 < f < 1.0
    c, f = O.voxel_of(0.0, 16, True)    # smoothstep half-voxel offset
    assert c == 0 and f == 0.5
    c, f = O.voxel_of(1.0, 16, True)    # capped at N(1-2^-20)
    assert c == 15
    c, f = O.voxel_of(-1e-7, 16, False)
    assert c == 0 and f == 0.0
