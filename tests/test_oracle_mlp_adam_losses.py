"""Pins the oracle's MLP, losses and Adam against the reference's own tests
(test_mlp.cpp, test_losses.cpp, test_adam.cpp; cited per test)."""
import math

import numpy as np
import pytest

import oracle as O
from _approx import approx_eq


# ---------------------------------------------------------------- MLP ----
def test_glorot_bounds_variance_zero_bias():   # test_mlp.cpp:10-36
    cfg = O.MlpCfg(64, 2, 64, 64)
    W, b = O.glorot_init(cfg, 123, np.float64)
    bound = math.sqrt(6.0 / 128)
    assert np.abs(W).max() <= bound
    assert W.size >= 10000
    assert abs(W.mean()) < 0.01
    assert approx_eq(W.var(), 2.0 / 128, 0.1)
    assert np.abs(b).max() == 0.0


def test_glorot_seed_deterministic():   # test_mlp.cpp:38-55
    cfg = O.MlpCfg(8, 1, 16, 4)
    a, _ = O.glorot_init(cfg, 5)
    b, _ = O.glorot_init(cfg, 5)
    c, _ = O.glorot_init(cfg, 6)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


def test_param_count(kats):   # test_mlp.cpp:57-67
    k = kats["mlp_param_count"]
    cfg = O.MlpCfg(32, 2, 64, 3)
    assert cfg.weight_count + cfg.bias_count == k["count"]
    assert len(cfg.layer_shapes()) == k["layers"]


def test_forward_matches_naive_loop():   # test_mlp.cpp:69-99
    cfg = O.MlpCfg(5, 2, 7, 2)
    W, b = O.glorot_init(cfg, 17, np.float64)
    rng = O.Pcg32(3, 0)
    X = np.array([rng.next_double() * 2 - 1 for _ in range(45)]).reshape(9, 5)
    out = O.mlp_forward(cfg, W, b, X)
    mats = O.split_weights(cfg, W)
    boff = np.cumsum([0] + [o for _, o in cfg.layer_shapes()])
    for s in range(9):
        a = X[s]
        for k, Wk in enumerate(mats):
            z = Wk @ a + b[boff[k]: boff[k + 1]]
            if k + 1 < len(mats):
                z = np.maximum(z, 0)
            a = z
        for i in range(2):
            assert approx_eq(out[s, i], a[i], 1e-13)


def test_sigmoid_output():   # test_mlp.cpp:101-125
    cfg = O.MlpCfg(3, 1, 8, 3, sigmoid=True)
    W, b = O.glorot_init(cfg, 2, np.float64)
    X = np.random.default_rng(0).uniform(-1, 1, (16, 3))
    out = O.mlp_forward(cfg, W, b, X)
    assert out.min() > 0 and out.max() < 1
    lin = O.mlp_forward(O.MlpCfg(3, 1, 8, 3, sigmoid=False), W, b, X)
    np.testing.assert_allclose(out, 1 / (1 + np.exp(-lin)), rtol=1e-13)


@pytest.mark.parametrize("sigmoid", [False, True])
def test_backward_finite_differences(sigmoid):   # test_mlp.cpp:127-197
    cfg = O.MlpCfg(4, 2, 6, 3, sigmoid=sigmoid)
    W, b = O.glorot_init(cfg, 31, np.float64)
    rng = O.Pcg32(8, 0)
    X = np.array([rng.next_double() * 2 - 1 for _ in range(20)]).reshape(5, 4)
    dOut = np.array([rng.next_double() * 2 - 1 for _ in range(15)]).reshape(5, 3)
    _, gW, gb, dX = O.mlp_forward_backward(cfg, W, b, X, dOut)

    def obj():
        return (dOut * O.mlp_forward(cfg, W, b, X)).sum()

    h = 1e-6
    for arr, grad, step in ((W, gW, 3), (b, gb, 2), (X, dX.ravel(), 4)):
        flat = arr.reshape(-1)
        for i in range(0, flat.size, step):
            save = flat[i]
            flat[i] = save + h
            fp = obj()
            flat[i] = save - h
            fm = obj()
            flat[i] = save
            assert approx_eq(grad.reshape(-1)[i], (fp - fm) / (2 * h), 1e-4)


def test_backward_accumulates():   # test_mlp.cpp:199-219
    cfg = O.MlpCfg(2, 1, 4, 1)
    W, b = O.glorot_init(cfg, 7, np.float64)
    X = np.random.default_rng(3).uniform(-1, 1, (3, 2))
    dOut = np.ones((3, 1))
    _, g1, _, _ = O.mlp_forward_backward(cfg, W, b, X, dOut)
    _, g2, gb2, _ = O.mlp_forward_backward(cfg, W, b, X, dOut)
    O.mlp_forward_backward(cfg, W, b, X, dOut, g2, gb2)
    assert np.abs(g2 - 2 * g1).max() < 1e-14


def test_forward_rejects_width():   # test_mlp.cpp:221-229
    cfg = O.MlpCfg(4, 2, 64, 3)
    W, b = O.glorot_init(cfg, 1)
    with pytest.raises(O.OracleInvalidArgument):
        O.mlp_forward(cfg, W, b, np.zeros((2, 3), np.float32))


# ------------------------------------------------------------- losses ----
def _fd_check(kind, p, t):   # test_losses.cpp:13-31
    _, dp = O.loss_with_grad(kind, p, t)
    h = 1e-7
    for i in range(p.size):
        q = p.copy().ravel()
        q[i] += h
        fp, _ = O.loss_with_grad(kind, q.reshape(p.shape), t)
        q[i] -= 2 * h
        fm, _ = O.loss_with_grad(kind, q.reshape(p.shape), t)
        assert approx_eq(dp.ravel()[i], (fp - fm) / (2 * h), 1e-5)


def test_l2_loss(kats):   # test_losses.cpp:35-55
    k = kats["l2"]
    loss, dp = O.loss_with_grad(O.LOSS_L2, np.array([k["pred"]]), np.array([k["target"]]))
    assert approx_eq(loss, k["loss"])
    np.testing.assert_allclose(dp[0], k["dpred"])
    t = np.array([k["target"]])
    loss, dp = O.loss_with_grad(O.LOSS_L2, t, t)
    assert loss == 0.0 and np.abs(dp).max() == 0.0
    rng = O.Pcg32(1, 0)
    p = np.array([rng.next_double() * 2 - 1 for _ in range(15)]).reshape(5, 3)
    t = np.array([rng.next_double() * 2 - 1 for _ in range(15)]).reshape(5, 3)
    _fd_check(O.LOSS_L2, p, t)


def test_mape_loss(kats):   # test_losses.cpp:57-89
    for c in kats["mape"]["cases"]:
        loss, dp = O.loss_with_grad(O.LOSS_MAPE, np.array([[c["pred"]]]), np.array([[c["target"]]]))
        if c["loss"] == 0.0:
            assert loss == 0.0
        else:
            assert approx_eq(loss, c["loss"])
        if "dpred" in c:
            if c["dpred"] == 0.0:
                assert dp[0, 0] == 0.0
            else:
                assert approx_eq(dp[0, 0], c["dpred"])
    rng = O.Pcg32(2, 0)
    p = np.array([rng.next_double() * 2 - 1 for _ in range(8)]).reshape(4, 2)
    t = np.array([rng.next_double() * 2 - 1 for _ in range(8)]).reshape(4, 2)
    _fd_check(O.LOSS_MAPE, p, t)


def test_relative_l2_frozen_denominator(kats):   # test_losses.cpp:91-106
    k = kats["relative_l2"]
    loss, dp = O.loss_with_grad(O.LOSS_REL_L2, np.array([[k["pred"]]]), np.array([[k["target"]]]))
    assert approx_eq(loss, k["loss"])
    assert approx_eq(dp[0, 0], k["dpred"])
    denom = 0.3 * 0.3 + 0.01
    full = (2.0 * 0.2 * denom - 0.04 * 2.0 * 0.3) / (denom * denom)
    assert not approx_eq(dp[0, 0], full)
    t = np.array([[k["target"]]])
    assert O.loss_with_grad(O.LOSS_REL_L2, t, t)[0] == 0.0


def test_psnr(kats):   # test_losses.cpp:108-123
    a = np.full((4, 4), 0.25, np.float32)
    assert O.psnr(a, a) == 100.0
    z = np.zeros((4, 4), np.float32)
    assert approx_eq(O.psnr(np.ones((4, 4), np.float32), z), 0.0)
    assert approx_eq(O.psnr(np.full((4, 4), 0.5, np.float32), z), 6.0206, 1e-4)
    assert O.psnr(np.full((4, 4), 1e-6, np.float32), z) <= 100.0


def test_loss_shape_mismatch():   # test_losses.cpp:125-132
    a, b = np.zeros((2, 3)), np.zeros((3, 2))
    for kind in (O.LOSS_L2, O.LOSS_MAPE, O.LOSS_REL_L2):
        with pytest.raises(O.OracleInvalidArgument):
            O.loss_with_grad(kind, a, b)
    with pytest.raises(O.OracleInvalidArgument):
        O.psnr(a, b)


# --------------------------------------------------------------- Adam ----
def _group(p, g, name="p", l2=False, skip=False):
    return O.ParamGroup(name, np.asarray(p, np.float64), np.asarray(g, np.float64), l2, skip)


def test_adam_first_step(kats):   # test_adam.cpp:26-46
    k = kats["adam_first_step"]
    g = _group(k["params"], k["grads"])
    st = O.AdamState()
    st.init([g])
    O.adam_step(st, [g], O.Hyper(lr=k["lr"]), k["lr"])
    for got, exp in zip(g.params, k["expected"]):
        assert approx_eq(got, exp, k["rel_eps"])
    assert (g.grads == 0).all()
    assert st.step == 1


def test_adam_skip_zero_bitwise():   # test_adam.cpp:48-90
    g = _group([1.0, 2.0, 3.0], [0.5, 0.0, -0.5], "tables", skip=True)
    st = O.AdamState()
    st.init([g])
    O.adam_step(st, [g], O.Hyper(), 1e-2)
    assert g.params[1] == 2.0 and st.m[0][1] == 0.0 and st.v[0][1] == 0.0
    assert g.params[0] != 1.0 and g.params[2] != 3.0
    plain = _group([1.0], [0.5])
    s2 = O.AdamState()
    s2.init([plain])
    O.adam_step(s2, [plain], O.Hyper(), 1e-2)
    after = plain.params[0]
    plain.grads[0] = 0.0
    O.adam_step(s2, [plain], O.Hyper(), 1e-2)
    assert plain.params[0] != after
    skip = _group([1.0], [0.5], "t", skip=True)
    s3 = O.AdamState()
    s3.init([skip])
    O.adam_step(s3, [skip], O.Hyper(), 1e-2)
    held = skip.params[0]
    skip.grads[0] = 0.0
    O.adam_step(s3, [skip], O.Hyper(), 1e-2)
    assert skip.params[0] == held


def test_adam_l2_flagged_only():   # test_adam.cpp:92-118
    hy = O.Hyper(lr=0.1, l2=0.5)
    w = _group([2.0], [0.0], "w", l2=True)
    s = O.AdamState()
    s.init([w])
    O.adam_step(s, [w], hy, 0.1)
    assert w.params[0] < 2.0
    b = _group([2.0], [0.0], "b")
    s = O.AdamState()
    s.init([b])
    O.adam_step(s, [b], hy, 0.1)
    assert b.params[0] == 2.0


def test_adam_bias_correction():   # test_adam.cpp:120-139
    g = _group([0.0], [1.0])
    s = O.AdamState()
    s.init([g])
    for i in range(500):
        g.grads[0] = 1.0
        before = g.params[0]
        O.adam_step(s, [g], O.Hyper(lr=0.01), 0.01)
        if i > 400:
            assert approx_eq(before - g.params[0], 0.01, 1e-3)
    assert s.step == 500


def test_adam_scale_invariance():   # test_adam.cpp:141-158
    d = []
    for scale in (1.0, 1000.0):
        g = _group([1.0], [0.37 * scale])
        s = O.AdamState()
        s.init([g])
        O.adam_step(s, [g], O.Hyper(lr=0.01), 0.01)
        d.append(1.0 - g.params[0])
    assert approx_eq(d[0], d[1], 1e-9)


def test_adam_nonfinite_names_group():   # test_adam.cpp:160-174
    g = _group([1.0], [float("nan")], "mlp_weights")
    s = O.AdamState()
    s.init([g])
    with pytest.raises(O.OracleRuntimeError, match="mlp_weights"):
        O.adam_step(s, [g], O.Hyper(), 1e-2)
    assert g.params[0] == 1.0 and s.step == 0


def test_lr_at(kats):   # test_adam.cpp:176-195
    k = kats["lr_at"]
    for step, lr in k["cases"]:
        assert approx_eq(O.lr_at(k["milestones"], k["factor"], k["base"], step), lr)
    prev = 1e9
    for step in range(0, 50001, 500):
        lr = O.lr_at(k["milestones"], k["factor"], k["base"], step)
        assert lr <= prev
        prev = lr


def test_default_schedule(kats):   # test_adam.cpp:197-213
    for total, ms in kats["default_schedule"]["cases"]:
        assert O.default_milestones(total) == ms


def test_hyper_defaults(kats):   # test_adam.cpp:227-235
    k = kats["adam_defaults"]
    h = O.Hyper()
    assert (h.beta1, h.beta2, h.eps, h.l2) == (k["beta1"], k["beta2"], k["eps"], k["l2"])


def test_adam_multi_span_contiguous():   # test_adam.cpp:237-256 (spans concatenated in one group)
    g = _group([1.0, 2.0, 3.0], [0.1, 0.2, 0.3], "multi")
    s = O.AdamState()
    s.init([g])
    O.adam_step(s, [g], O.Hyper(), 1e-2)
    assert approx_eq(s.m[0][2], 0.1 * 0.3)
    assert g.params[2] < 3.0
