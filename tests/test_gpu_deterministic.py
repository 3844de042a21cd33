"""Deterministic-backward option (nfg_options.deterministic; "a
strictly single-threaded deterministic mode must exist for tests").

* encode_backward: for identical dY the table gradients are BIT-IDENTICAL to
  the reference's single-threaded loop (grid.hpp:286-294: level -> point ->
  corner, grad += w * dY in fp32), because every row receives the same
  sequence of round-to-nearest additions (sorted per-row reduction).
* train_step / gradients / mlp_backward: run-to-run bit-reproducible (MLP
  partials and the loss sum reduced in a fixed CTA order), and within the
  usual fp16-MMA tolerance of the default (atomic) path.
"""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import ENC_CASES, _grid, _model, _nf, _ocfg, _points

pytestmark = pytest.mark.gpu


def _det_model(nf, g, **kw):
    m = nf.FieldModel(options=nf.Options(table_fp32=kw.pop("table_fp32", True), deterministic=True))
    m.hash_cfg = g
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=kw.pop("n_out", 1))
    m.hyper = nf.AdamHyper(lr=kw.pop("lr", 1e-3))
    m.init(kw.pop("seed", 1337))
    return m


@pytest.mark.parametrize("case", ENC_CASES)
def test_encode_backward_bit_exact_in_reference_order(case):   # grid.hpp:277-295
    nf = _nf()
    g = _grid(nf, **case)
    m = _det_model(nf, g)
    og = _ocfg(g)
    want = np.zeros(m.sizes[0], np.float32)
    for seed in (11, 12):   # two calls: gradients accumulate (+=) in call order
        X = _points(3001, g.dims, seed=seed)
        X[:3] = [[0.0] * g.dims, [1.0] * g.dims, [0.5] * g.dims]
        dY = O.Pcg32(seed, 3).floats(3001 * g.levels * g.features).reshape(3001, -1) * 2 - 1
        m.encode_backward(X, dY)
        _, cache = O.encode_forward(og, m.table_params, X)
        O.encode_backward(og, cache, dY, want)
    got = m.grads[: m.sizes[0]]
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_train_steps_bit_reproducible_and_close_to_default_path():   # model.cpp:111-138
    nf = _nf()
    g = _grid(nf, dims=3, levels=16, table_size=1 << 16, features=2, n_min=16, n_max=1024)
    runs = []
    for _ in range(2):
        m = _det_model(nf, g, table_fp32=False)
        rng = O.Pcg32(21, 4)
        losses = []
        for step in range(1, 4):
            X = rng.floats(20000 * 3).reshape(20000, 3)
            T = O.csg_sdf(X).reshape(-1, 1)
            losses.append(m.train_step(X, T, nf.LossKind.Mape, step))
        runs.append((losses, m.params, m.adam_state()))
    (l0, p0, s0), (l1, p1, s1) = runs
    assert l0 == l1
    assert np.array_equal(p0.view(np.uint32), p1.view(np.uint32))
    for a, b in zip(s0[1:], s1[1:]):
        assert np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))
    # the default (atomic, fused) path agrees within the parity tolerance
    m = _model(nf, g, lr=1e-3)
    rng = O.Pcg32(21, 4)
    for step in range(1, 4):
        X = rng.floats(20000 * 3).reshape(20000, 3)
        T = O.csg_sdf(X).reshape(-1, 1)
        lf = m.train_step(X, T, nf.LossKind.Mape, step)
        assert abs(lf - l0[step - 1]) <= 1e-3 * abs(l0[step - 1])


def test_mlp_backward_and_gradients_reproducible():   # mlp.hpp:129-158
    nf = _nf()
    g = _grid(nf, dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=1024)
    outs = []
    for _ in range(2):
        m = _det_model(nf, g, n_out=3)
        rng = O.Pcg32(5, 5)
        Y = rng.floats(5000 * 32).reshape(5000, 32) * 2 - 1
        dO = rng.floats(5000 * 3).reshape(5000, 3) - 0.5
        dY = m.mlp_backward(Y, dO)
        X = rng.floats(5000 * 2).reshape(5000, 2)
        loss = m.gradients(X, rng.floats(5000 * 3).reshape(5000, 3), nf.LossKind.L2)
        outs.append((dY, loss, m.grads))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][2].view(np.uint32), outs[1][2].view(np.uint32))
