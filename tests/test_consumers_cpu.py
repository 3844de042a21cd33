"""Oracle restatements of the inference consumers (tasks.cpp:195-356) against
the reference's own test cases (test_tasks.cpp:108-205), CPU only."""
import math

import numpy as np
import pytest

import oracle as O

CAM = dict(position=(0.5, 0.5, -1.2), target=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0), fov_deg=40.0)


def sphere(X):   # test_tasks.cpp:158-166
    p = X.astype(np.float64)
    return (np.sqrt(((p - 0.5) ** 2).sum(1)) - 0.25).astype(np.float32)


def test_oracle_render_sphere_silhouette():   # test_tasks.cpp:155-199
    W = H = 64
    img = O.render_sdf_shaded(sphere, W=W, H=H, **CAM)
    px = lambda x, y: img[y * W + x]   # noqa: E731
    assert px(1, 1)[0] == pytest.approx(1.0)
    assert 0.0 < px(W // 2, H // 2)[0] < 1.0
    dist = math.sqrt(0.0 + 0.0 + 1.7 ** 2)
    focal = 0.5 * H / math.tan(0.5 * 40.0 * math.pi / 180.0)
    expected = focal * math.tan(math.asin(0.25 / dist))
    row = [x for x in range(W) if px(x, H // 2)[0] < 0.999]
    assert row
    assert 0.5 * (row[-1] - row[0] + 1) == pytest.approx(expected, rel=0.12)
    blank = O.render_sdf_shaded(lambda X: np.full(X.shape[0], 0.5, np.float32), W=16, H=16, **CAM)
    assert blank.min() == pytest.approx(1.0)


def test_oracle_iou_boxes():   # test_tasks.cpp:108-142
    model = lambda X: np.where(X[:, 0] < 0.6, -1.0, 1.0)   # noqa: E731
    v = O.iou(model, lambda p: -1 if p[0] > 0.4 else 1, 1 << 16, O.Pcg32(1, 0))
    assert v == pytest.approx(0.2, rel=0.05)
    assert O.iou(model, lambda p: -1 if p[0] < 0.6 else 1, 1 << 12, O.Pcg32(1, 0)) == 1.0
    assert O.iou(model, lambda p: -1 if p[0] > 0.9 else 1, 1 << 12, O.Pcg32(1, 0)) < 0.01
    assert O.iou(lambda X: np.ones(X.shape[0]), lambda p: 1, 1024, O.Pcg32(1, 0)) == 1.0
