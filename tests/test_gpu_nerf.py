"""NeRF on the device (BASELINE config 4) against the
restatement of the paper's appendix (oracle; parity UNPINNED — the reference
has no NeRF):

* occupancy-grid marching + compaction: sample counts and positions
  bit-identical (fp32 in the same operation order);
* compositing forward/backward, SH4, and the synthetic scene renderer within
  stated fp32 tolerances;
* training on the synthetic scene converges (loss and held-out PSNR) and the
  occupancy grid culls empty space.
"""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import _nf

pytestmark = pytest.mark.gpu


def _random_bits(seed=1, frac=0.3):
    rng = np.random.default_rng(seed)
    # blocky occupancy: 8^3-cell blocks on/off, in Morton order
    blocks = rng.uniform(size=(16, 16, 16)) < frac
    x, y, z = np.meshgrid(np.arange(128), np.arange(128), np.arange(128), indexing="ij")
    on = blocks[x // 8, y // 8, z // 8].ravel()
    m = O.morton3(x.ravel(), y.ravel(), z.ravel())
    bits = np.zeros(128 ** 3 // 8, np.uint8)
    np.bitwise_or.at(bits, m[on] >> 3, (1 << (m[on] & 7)).astype(np.uint8))
    return bits


def _rays(n, seed=2):
    rng = np.random.default_rng(seed)
    o = rng.uniform(-0.5, 1.5, (n, 3))
    target = rng.uniform(0.2, 0.8, (n, 3))
    d = target - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = np.concatenate([o, d], axis=1).astype(np.float32)
    rays[:4, :3] = [[0.5, 0.5, 0.5], [0.0, 0.0, 0.0], [0.25, 0.75, -1.0], [0.5, 0.5, 2.0]]   # inside / corner / axis
    rays[2, 3:] = [0.0, 0.0, 1.0]
    rays[3, 3:] = [0.0, 0.0, -1.0]
    return rays


def test_march_compaction_bit_exact():
    nf = _nf()
    rays = _rays(300)
    for bits in (_random_bits(1, 0.3), np.full(128 ** 3 // 8, 255, np.uint8), _random_bits(5, 0.05)):
        counts, samples = nf.nerf_march(rays, bits, 1024)
        c_ref, s_ref = O.nerf_march(rays, bits, 1024)
        assert np.array_equal(counts, c_ref)
        assert np.array_equal(samples.view(np.uint32), s_ref.view(np.uint32))
    counts, _ = nf.nerf_march(rays, np.full(128 ** 3 // 8, 255, np.uint8), 64)   # per-ray cap
    assert counts.max() == 64


def test_composite_forward_backward():
    nf = _nf()
    rng = np.random.default_rng(4)
    counts = rng.integers(0, 40, 257).astype(np.uint32)
    counts[:3] = [0, 1, 300]
    S = int(counts.sum())
    raw = rng.normal(4.0, 2.0, S).astype(np.float32)
    raw[-300:] = 9.0   # opaque run: transmittance stop
    rgb = rng.uniform(0, 1, (S, 3)).astype(np.float32)
    tgt = rng.uniform(0, 1, (257, 3)).astype(np.float32)
    col, d_rgb, d_raw, loss = nf.nerf_composite(counts, raw, rgb, tgt, (1.0, 0.5, 0.0))
    col_r, d_rgb_r, d_raw_r, loss_r = O.nerf_composite(counts, raw, rgb, tgt, (1.0, 0.5, 0.0))
    assert np.abs(col - col_r).max() <= 2e-5
    assert abs(loss - loss_r) <= 1e-4 * loss_r
    assert np.abs(d_rgb - d_rgb_r).max() <= 1e-5 * np.abs(d_rgb_r).max() + 1e-9
    assert np.abs(d_raw - d_raw_r).max() <= 1e-3 * np.abs(d_raw_r).max() + 1e-9


def test_sh4():
    nf = _nf()
    rng = np.random.default_rng(7)
    d = rng.normal(size=(5000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    assert np.abs(nf.nerf_sh4(d.astype(np.float32)) - O.sh4(d.astype(np.float32))).max() <= 2e-6


def test_scene_render_matches_oracle():
    nf = _nf()
    cams, focal = nf.orbit_cameras(2, width=32)
    img = nf.nerf_scene_render(cams, 32, 24, focal)
    for v in range(2):
        ref = O.nerf_scene_render(cams[v], 32, 24, focal)
        assert np.abs(img[v] - ref).max() <= 2e-3
        assert np.abs(img[v] - ref).mean() <= 1e-4


def test_nerf_training_converges_and_culls():   # BASELINE config 4 shape at desk scale
    nf = _nf()
    W = H = 64
    cams, focal = nf.orbit_cameras(12, width=W)
    images = nf.nerf_scene_render(cams, W, H, focal)
    held_cam, _ = nf.orbit_cameras(1, width=W, phase=0.37)
    held = nf.nerf_scene_render(held_cam, W, H, focal)[0]
    nerf = nf.NeRF(grid=nf.HashEncodingConfig(levels=16, table_size=1 << 17, features=2, n_min=16, n_max=512, dims=3),
                   lr=1e-2, target_samples=1 << 16, seed=3)
    nerf.set_dataset(cams, images, W, H, focal)
    losses = []
    for step in range(1, 401):
        loss, nr, ns = nerf.train_step(step)
        assert 0 < ns <= 1 << 16 and nr > 0
        losses.append(loss)
    assert np.mean(losses[-20:]) < 0.2 * np.mean(losses[:5])
    pred = nerf.render(held_cam[0], W, H, focal)
    psnr = -10 * np.log10(np.mean((pred - held) ** 2))
    assert psnr > 20.0, psnr
    bits, dens = nerf.occupancy()
    occupied = np.unpackbits(bits).mean()
    assert occupied < 0.5, occupied   # empty space is skipped
    # the scene's spheres are occupied
    c = [O.morton3(int(0.40 * 128), int(0.45 * 128), int(0.50 * 128))]
    assert (bits[c[0] >> 3] >> (c[0] & 7)) & 1


def test_field_backward_device_fused_matches_staged():   # nfg_field_backward_device (density network)
    nf = _nf()
    import torch
    g = nf.HashEncodingConfig(levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512, dims=3)
    grads = []
    for fused in (True, False):
        m = nf.FieldModel(options=nf.Options(table_fp32=True, fused_train=fused))
        m.hash_cfg = g
        m.mlp_cfg = nf.MlpConfig(hidden_layers=1, hidden_width=64, output_width=16)
        m.init(5)
        rng = O.Pcg32(5, 5)
        X = torch.from_numpy(rng.floats(4000 * 3).reshape(4000, 3)).cuda()
        dO = torch.from_numpy(rng.floats(4000 * 16).reshape(4000, 16) - 0.5).cuda() * 1e-3
        from paper_2201_05989_b200 import _lib as L
        L.check(m.lib.nfg_field_backward_device(m.h, X.data_ptr(), 4000, dO.data_ptr()))
        m.check()
        grads.append(m.grads)
    a, b = grads
    assert np.array_equal(a != 0, b != 0)
    assert np.linalg.norm(a - b) <= 2e-2 * np.linalg.norm(b)


def test_backward_compaction_path(monkeypatch):   # second compaction: only pre-stop samples reach the backward
    nf = _nf()
    W = H = 48
    cams, focal = nf.orbit_cameras(8, width=W)
    images = nf.nerf_scene_render(cams, W, H, focal)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("NFG_NERF_COMPACT", mode)
        nerf = nf.NeRF(grid=nf.HashEncodingConfig(levels=16, table_size=1 << 16, features=2, n_min=16, n_max=256,
                                                  dims=3),
                       lr=1e-2, target_samples=1 << 15, background=(0.0, 0.0, 0.0), seed=5)
        nerf.set_dataset(cams, images, W, H, focal)
        losses = [nerf.train_step(s)[0] for s in range(1, 151)]
        res[mode] = (np.mean(losses[:5]), np.mean(losses[-10:]), nerf.last_backward_samples)
    for first, last, nb in res.values():
        assert last < 0.3 * first and nb > 0
    assert abs(res["0"][1] - res["1"][1]) <= 0.5 * res["0"][1]
