"""Inference consumers on the device (tasks.cpp:195-356):
render_image, render_sdf_shaded (sphere tracing with active-ray compaction)
and iou, against the oracle restatements on the SAME field function — the ray
and point arithmetic is double precision in the reference's order on both
sides, so images and IoU values are compared exactly."""
import math

import numpy as np
import pytest

import oracle as O
from test_consumers_cpu import CAM, sphere
from test_gpu_parity import _nf

pytestmark = pytest.mark.gpu


def _cam(nf):
    return nf.Camera(**CAM)


def _sdf_model(nf, steps=60):
    m = nf.FieldModel()
    m.hash_cfg = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 16, features=2, n_min=16, n_max=512)
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
    m.hyper = nf.AdamHyper(lr=1e-2)
    m.init(7)
    rng = O.Pcg32(7, 2)
    for step in range(1, steps + 1):
        X = rng.floats(3 * (1 << 14)).reshape(-1, 3)
        m.train_step(X, O.csg_sdf(X).reshape(-1, 1), nf.LossKind.L2, step)
    return m


def test_render_image_constant_and_exact():   # test_tasks.cpp:145-153, tasks.cpp:195-209
    nf = _nf()
    m = nf.FieldModel()
    m.hash_cfg = nf.HashEncodingConfig(dims=2, levels=4, table_size=1 << 10, features=2, n_min=4, n_max=32)
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=3,
                             output_activation=nf.OutputActivation.Sigmoid)
    m.init(1)
    t, w, b = m.sizes
    p = m.params
    p[t:] = 0.0   # constant model: sigmoid(0)
    m.write(0, p)
    img = nf.render_image(m, 16, 8)
    assert img.shape == (128, 3) and np.all(img == 0.5)
    m.init(2)
    img = nf.render_image(m, 33, 17)
    x = np.arange(33 * 17)
    X = np.stack([((x % 33).astype(np.float32) + np.float32(0.5)) / np.float32(33),
                  ((x // 33).astype(np.float32) + np.float32(0.5)) / np.float32(17)], axis=1)
    assert np.array_equal(img, m.evaluate(X))


def test_render_sdf_shaded_analytic_sphere_matches_oracle():   # test_tasks.cpp:155-199
    nf = _nf()
    W = H = 64
    img = nf.render_sdf_shaded(sphere, _cam(nf), W, H)
    ref = O.render_sdf_shaded(sphere, W=W, H=H, **CAM)
    assert np.array_equal(img, ref)
    row = [x for x in range(W) if img[(H // 2) * W + x][0] < 0.999]
    focal = 0.5 * H / math.tan(0.5 * 40.0 * math.pi / 180.0)
    expected = focal * math.tan(math.asin(0.25 / 1.7))
    assert 0.5 * (row[-1] - row[0] + 1) == pytest.approx(expected, rel=0.12)
    blank = nf.render_sdf_shaded(lambda X: np.full(X.shape[0], 0.5, np.float32), _cam(nf), 16, 16)
    assert blank.min() == 1.0


def test_render_sdf_shaded_trained_model_matches_oracle_tracer():   # device field, compaction on the GPU
    nf = _nf()
    m = _sdf_model(nf)
    W, H = 96, 80
    img = nf.render_sdf_shaded(m, _cam(nf), W, H)
    ref = O.render_sdf_shaded(lambda X: m.evaluate(X), W=W, H=H, **CAM)
    assert np.array_equal(img, ref)
    assert (img[:, 0] < 0.999).sum() > 100   # the torus/sphere is visible


def test_iou_matches_oracle_and_reference_boxes():   # test_tasks.cpp:108-142, tasks.cpp:331-356
    nf = _nf()
    model = lambda X: np.where(X[:, 0] < 0.6, -1.0, 1.0).astype(np.float32)   # noqa: E731
    inside = lambda p: -1 if p[0] > 0.4 else 1   # noqa: E731
    v = nf.iou(model, inside, 1 << 16, nf.DeviceRng(1, 0))
    assert v == O.iou(model, inside, 1 << 16, O.Pcg32(1, 0))
    assert v == pytest.approx(0.2, rel=0.05)
    assert nf.iou(model, lambda p: -1 if p[0] < 0.6 else 1, 1 << 12, nf.DeviceRng(1, 0)) == 1.0
    assert nf.iou(lambda X: np.ones(X.shape[0], np.float32), lambda p: 1, 1024, nf.DeviceRng(1, 0)) == 1.0
    # trained device model vs the analytic CSG interior, chunked (> 2^16 points), continuing streams
    m = _sdf_model(nf)
    csg = lambda p: -1 if O.csg_sdf(p.reshape(1, 3).astype(np.float32))[0] < 0 else 1   # noqa: E731
    r_d, r_h = nf.DeviceRng(11, 11), O.Pcg32(11, 11)
    for n in (70000, 1000):
        a = nf.iou(m, csg, n, r_d, (0.1, 0.1, 0.1), (0.9, 0.9, 0.9))
        b = O.iou(lambda X: m.evaluate(X), csg, n, r_h, (0.1, 0.1, 0.1), (0.9, 0.9, 0.9))
        assert a == b
    assert a > 0.3
