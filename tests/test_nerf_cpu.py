"""NeRF restatement (oracle; parity UNPINNED — the reference has no NeRF,
SPEC.md:8): self-consistency of the paper-appendix restatement on CPU."""
import numpy as np

import oracle as O


def test_march_full_and_empty_grid():
    rays = np.array([[0.5, 0.5, -1.0, 0.01, 0.02, 1.0], [0.2, 0.3, 2.0, 0.0, 0.0, -1.0],
                     [-1.0, -1.0, -1.0, -1.0, 0.0, 0.0]], np.float32)
    rays[:, 3:] /= np.linalg.norm(rays[:, 3:], axis=1, keepdims=True)
    full = np.full(128 ** 3 // 8, 255, np.uint8)
    c, s = O.nerf_march(rays, full)
    assert c[2] == 0                                   # misses the cube
    assert abs(int(c[1]) - round(1.0 / float(O.NERF_DT))) <= 1   # straight through, dt = sqrt(3)/1024
    assert np.all((s >= 0) & (s <= 1))
    c, s = O.nerf_march(rays, np.zeros_like(full))
    assert c.sum() == 0 and len(s) == 0                # empty grid: every step skipped


def test_march_skips_only_empty_cells():
    bits = np.zeros(128 ** 3 // 8, np.uint8)
    for x in range(60, 70):                            # a 10^3 block of occupied cells
        for y in range(60, 70):
            for z in range(60, 70):
                m = O.morton3(x, y, z)
                bits[m >> 3] |= 1 << (m & 7)
    ray = np.array([[0.51, 0.52, -0.5, 0.0, 0.0, 1.0]], np.float32)
    c, s = O.nerf_march(ray, bits)
    assert c[0] > 0
    cells = np.floor(s * 128).astype(int)
    assert np.all((cells >= 60) & (cells < 70))
    assert abs(int(c[0]) - round((10 / 128) / float(O.NERF_DT))) <= 2


def test_composite_gradients_finite_difference():
    rng = np.random.default_rng(3)
    counts = np.array([5, 0, 9, 3], np.uint32)
    S = int(counts.sum())
    raw = rng.normal(3.0, 1.5, S)
    rgb = rng.uniform(0, 1, (S, 3))
    tgt = rng.uniform(0, 1, (4, 3))
    _, d_rgb, d_raw, L0 = O.nerf_composite(counts, raw, rgb, tgt, dt=0.05)
    L = lambda rw, c: O.nerf_composite(counts, rw, c, tgt, dt=0.05)[3] / 12.0   # noqa: E731  (mean over rays x 3)
    h = 1e-6
    for i in range(S):
        e = np.zeros(S)
        e[i] = h
        fd = (L(raw + e, rgb) - L(raw - e, rgb)) / (2 * h)
        assert abs(fd - d_raw[i]) <= 1e-5 * max(1.0, abs(fd)), (i, fd, d_raw[i])
        for k in range(3):
            E = np.zeros_like(rgb)
            E[i, k] = h
            fd = (L(raw, rgb + E) - L(raw, rgb - E)) / (2 * h)
            assert abs(fd - d_rgb[i, k]) <= 1e-5 * max(1.0, abs(fd))


def test_sh4_orthonormal():   # the 16 real SH basis functions are orthonormal on the sphere
    rng = np.random.default_rng(0)
    d = rng.normal(size=(200000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    Y = O.sh4(d)
    G = 4 * np.pi * (Y.T @ Y) / len(d)
    assert np.abs(G - np.eye(16)).max() < 0.03
