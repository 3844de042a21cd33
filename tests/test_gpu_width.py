"""Hidden widths below 64 (mlp.hpp:15-40 allows any width; the reference's own
tests use 4, 8 and 16, e.g. acceptance.cpp:337). The sm_100a kernels run the
64-wide tensor-core layers with zero rows / columns beyond the width: padded
units have z = 0, ReLU(0) = 0 and a zero dz, so the real units' forward and
backward are those of the narrow MLP (exact zeros added in fp32).
Tolerances as test_gpu_parity.test_train_step_parity (fp32 tables)."""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import _grid, _ocfg, _points

pytestmark = pytest.mark.gpu


def _pair(nf, g, hw, hl, n_out, sig, fused=True, engine=0, lr=1e-3):
    m = nf.FieldModel(options=nf.Options(table_fp32=True, fused_train=fused, mlp_engine=engine))
    m.hash_cfg = g
    m.mlp_cfg = nf.MlpConfig(hidden_layers=hl, hidden_width=hw, output_width=n_out,
                             output_activation=nf.OutputActivation.Sigmoid if sig else nf.OutputActivation.Linear)
    m.hyper = nf.AdamHyper(lr=lr)
    m.init(1337)
    f = O.Field(_ocfg(g), O.MlpCfg(hidden_layers=hl, hidden_width=hw, output_width=n_out, sigmoid=sig),
                O.Hyper(lr=lr))
    f.init(1337)
    return m, f


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("hw,hl", [(8, 1), (16, 2), (32, 2), (48, 3), (4, 1)])
def test_narrow_mlp_train_parity(hw, hl, fused):
    from paper_2201_05989_b200 import nf
    g = _grid(nf, dims=3, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512)
    n_out, sig, kind = 1, False, 1
    m, f = _pair(nf, g, hw, hl, n_out, sig, fused=fused)
    assert m.parameter_count() == f.params.size
    assert np.array_equal(m.params, f.params)   # PCG32 tables + Glorot at width hw, bit-exact
    t, w, _ = m.sizes
    rng = O.Pcg32(21, 4)
    X = rng.floats(3000 * 3).reshape(3000, 3)
    T = rng.floats(3000).reshape(3000, 1) * 0.6 - 0.3
    lg = m.gradients(X, T, kind)
    G = m.grads
    og = _ocfg(g)
    mc = O.MlpCfg(g.levels * g.features, hl, hw, n_out, sig)
    P = m.params
    Y, cache = O.encode_forward(og, P[:t], X)
    pred = O.mlp_forward(mc, P[t:t + w], P[t + w:], Y)
    lo, dp = O.loss_with_grad(kind, pred, T)
    _, gW, gb, dY = O.mlp_forward_backward(mc, P[t:t + w], P[t + w:], Y, dp)
    gt = np.zeros(t, np.float32)
    O.encode_backward(og, cache, dY, gt)
    assert abs(lg - lo) <= 1e-4 * abs(lo)
    # same touched-entry set, up to entries below 1e-4 of the largest gradient
    # (an fp32 dY of exactly zero against an fp16-operand noise-floor value)
    import _fp16ref as R
    _, bad = R.touched_set_unexplained(G[:t], gt, gt)
    assert bad.size == 0, (bad[:10], G[:t][bad[:10]], gt[bad[:10]])
    for a, r in ((G[:t], gt), (G[t:t + w], gW), (G[t + w:], gb)):
        assert np.linalg.norm(a - r) <= 6e-2 * np.linalg.norm(r)
    m.write(1, np.zeros_like(G))
    for step in range(1, 4):
        X = rng.floats(3000 * 3).reshape(3000, 3)
        T = rng.floats(3000).reshape(3000, 1) * 0.6 - 0.3
        lg = m.train_step(X, T, kind, step)
        lo = f.train_step(X, T, kind, step)
        assert abs(lg - lo) <= 1e-3 * abs(lo) + 1e-7, (step, lg, lo)


@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("hw", [8, 32])
def test_narrow_mlp_evaluate(hw, engine):
    from paper_2201_05989_b200 import nf
    g = _grid(nf, dims=2, levels=16, table_size=1 << 12, features=2, n_min=16, n_max=256)
    m, f = _pair(nf, g, hw, 2, 3, True, engine=engine)
    rng = O.Pcg32(3, 3)
    for step in range(1, 4):
        X = rng.floats(4096 * 2).reshape(-1, 2)
        m.train_step(X, np.tile(X[:, :1], (1, 3)), nf.LossKind.L2, step)
    f.params[:] = m.params
    X = _points(5000, 2, seed=9)
    out = m.evaluate(X)
    ref = f.evaluate(X)
    assert np.abs(out - ref).max() <= 2e-3 * np.abs(ref).max() + 1e-5


def test_criterion4_zero_grad_skip_width8():   # acceptance.cpp:323-369, the reference's own shape (width 8)
    """Feature-table entries untouched by a batch stay bit-identical after a
    full training step; touched entries move."""
    from paper_2201_05989_b200 import nf
    g = nf.HashEncodingConfig(dims=2, levels=2, table_size=1 << 10, n_min=8, n_max=16, features=2)
    m = nf.FieldModel()
    m.hash_cfg = g
    m.mlp_cfg = nf.MlpConfig(hidden_layers=1, hidden_width=8, output_width=1)
    m.init(3)
    before = m.params
    X = np.array([[0.1, 0.1], [0.11, 0.11], [0.12, 0.12], [0.13, 0.13]], np.float32)
    T = np.full((4, 1), 0.3, np.float32)
    m.train_step(X, T, nf.LossKind.L2, 1)
    after = m.params
    t = m.sizes[0]
    og = _ocfg(g)
    _, cache = O.encode_forward(og, before[:t], X)
    specs = O.level_resolutions(og)
    touched = np.zeros(t // 2, bool)
    for l in range(g.levels):
        touched[specs[l].row_offset + cache.rows[l].ravel().astype(np.int64)] = True
    changed = np.any((after[:t] != before[:t]).reshape(-1, 2), axis=1)
    assert not changed[~touched].any()   # untouched table entries are bit-identical
    assert changed[touched].any()        # touched table entries actually move
