"""tcgen05 MLP engine (nfg_options.mlp_engine = NFG_MMA_TCGEN05) against the
mma.sync engine and the CPU oracle on identical parameters and inputs.

Both engines feed the tensor cores the same fp16 operands (encoded features,
weights, hidden activations) and accumulate in fp32; only the order of the
fp32 accumulation differs (one M=128 tcgen05.mma per K16 step vs m16n8k16
fragments), so a hidden activation may round to the neighbouring fp16 value.
Tolerance: |tc - sync| <= 1e-3 max|out| + 1e-5 (fp16 half-ulp flips propagated
through <= 3 layers); against the fp32 oracle the contract of
test_gpu_parity.test_evaluate_parity (mlp.hpp:104-124, model.cpp:102-109).
"""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import _grid, _model, _oracle_field, _points

pytestmark = pytest.mark.gpu

SYNC, TC = 1, 2


def _pair(nf, grid, hidden_layers=2, n_out=1, sigmoid=False, table_fp32=False, train_steps=3):
    ms = []
    for eng in (SYNC, TC):
        m = nf.FieldModel(options=nf.Options(table_fp32=table_fp32, mlp_engine=eng))
        m.hash_cfg = grid
        m.mlp_cfg = nf.MlpConfig(hidden_layers=hidden_layers, hidden_width=64, output_width=n_out,
                                 output_activation=nf.OutputActivation.Sigmoid if sigmoid
                                 else nf.OutputActivation.Linear)
        m.hyper = nf.AdamHyper(lr=1e-2)
        m.init(1337)
        ms.append(m)
    # a few training steps on the first model so the tables carry signal, then
    # copy the parameters into the second one
    rng = O.Pcg32(2, 2)
    d = grid.dims
    for step in range(1, train_steps + 1):
        X = rng.floats(8192 * d).reshape(-1, d)
        T = np.tile(O.csg_sdf(X if d == 3 else np.c_[X, X[:, :1]]).reshape(-1, 1), (1, n_out))
        ms[0].train_step(X, T.astype(np.float32), nf.LossKind.L2, step)
    ms[1].write(nf.BUF_PARAMS, ms[0].params)
    return ms


CASES = [
    dict(grid=dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048), hl=2, n_out=1),
    dict(grid=dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048), hl=1, n_out=1),
    dict(grid=dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048), hl=3, n_out=1),
    dict(grid=dict(dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=1024), hl=2, n_out=3,
         sigmoid=True),
    dict(grid=dict(dims=3, levels=8, table_size=1 << 14, features=2, n_min=16, n_max=256), hl=2, n_out=16),
    dict(grid=dict(dims=3, levels=16, table_size=1 << 16, features=2, n_min=16, n_max=512), hl=2, n_out=1,
         fp32=True),
    dict(grid=dict(dims=3, levels=8, table_size=1 << 14, features=4, n_min=16, n_max=256), hl=2, n_out=1),
    dict(grid=dict(dims=2, levels=32, table_size=1 << 12, features=1, n_min=4, n_max=512), hl=2, n_out=1),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_tc_engine_matches_sync(case):
    from paper_2201_05989_b200 import nf
    c = CASES[case]
    g = _grid(nf, **c["grid"])
    ms, mt = _pair(nf, g, hidden_layers=c["hl"], n_out=c["n_out"], sigmoid=c.get("sigmoid", False),
                   table_fp32=c.get("fp32", False))
    for B in (1, 100, 128, 129, 5000, (1 << 16) + 3):
        X = _points(B, g.dims, seed=B)
        a = ms.evaluate(X)
        assert "mma=tcgen05" not in ms.last_kernel_variant(1)
        b = mt.evaluate(X)
        assert "k_infer_tc" in mt.last_kernel_variant(1) and "mma=tcgen05" in mt.last_kernel_variant(1)
        assert a.shape == b.shape
        assert np.all(np.isfinite(b))
        err = np.abs(a - b).max()
        assert err <= 1e-3 * np.abs(a).max() + 1e-5, (B, err, np.abs(a).max())


def test_tc_engine_oracle_parity_config2():   # model.cpp:102-109 at config 2 through the tcgen05 engine
    from paper_2201_05989_b200 import nf
    g = _grid(nf, dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)
    m = nf.FieldModel(options=nf.Options(mlp_engine=TC))
    m.hash_cfg = g
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
    m.hyper = nf.AdamHyper(lr=1e-2)
    m.init(1337)
    f = _oracle_field(m)
    rng = O.Pcg32(2, 2)
    for step in range(1, 6):
        X = rng.floats(30000).reshape(-1, 3)
        m.train_step(X, O.csg_sdf(X).reshape(-1, 1), nf.LossKind.Mape, step)
    P = m.params
    nt = m.sizes[0]
    P[:nt] = P[:nt].astype(np.float16).astype(np.float32)   # the kernel gathers the fp16 shadow
    f.params[:] = P
    X = _points(1 << 16, 3, seed=77)
    out = m.evaluate(X)
    assert "mma=tcgen05" in m.last_kernel_variant(1)
    ref = f.evaluate(X)
    assert np.abs(out - ref).max() <= 2e-3 * np.abs(ref).max() + 1e-5


def test_tc_engine_empty_batch():
    from paper_2201_05989_b200 import nf
    g = _grid(nf, dims=3, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=256)
    ms, mt = _pair(nf, g, train_steps=0)
    out = mt.evaluate(np.zeros((0, 3), np.float32))
    assert out.shape[0] == 0


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("case", ["config2", "config1"])
def test_train_dw_engines_agree(case, det):   # model.cpp:111-138, dW on tcgen05 vs mma.sync
    """The fused step's dW / db reductions on tcgen05 (TMEM accumulators over
    all tiles of a CTA, rescaled to each tile's power-of-two dz scale) against the mma.sync
    reductions (register accumulators, per-tile scale): same fp16 operands, fp32
    accumulation in a different order; the bias gradients of the output layer
    come from the same fp16 dz in both."""
    from paper_2201_05989_b200 import nf
    if case == "config2":
        g = _grid(nf, dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)
        n_out, sig, kind = 1, False, nf.LossKind.Mape
    else:
        g = _grid(nf, dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=1024)
        n_out, sig, kind = 3, True, nf.LossKind.L2
    ms = []
    for eng in (SYNC, TC):
        m = nf.FieldModel(options=nf.Options(mlp_engine=eng, deterministic=det))
        m.hash_cfg = g
        m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=n_out,
                                 output_activation=nf.OutputActivation.Sigmoid if sig else nf.OutputActivation.Linear)
        m.hyper = nf.AdamHyper(lr=1e-3)
        m.init(1337)
        ms.append(m)
    rng = O.Pcg32(5, 5)
    d = g.dims
    for step in range(1, 4):   # move off the init with the tcgen05 model, then share its parameters
        X = rng.floats(16384 * d).reshape(-1, d)
        T = np.tile(O.csg_sdf(X if d == 3 else np.c_[X, X[:, :1]]).reshape(-1, 1), (1, n_out))
        if sig:
            T = np.clip(T + 0.5, 0, 1)
        ms[1].train_step(X, T.astype(np.float32), kind, step)
    ms[0].write(nf.BUF_PARAMS, ms[1].params)
    B = 3 * 65536 + 77   # several tiles per CTA (running scale) and a ragged tail
    X = rng.floats(B * d).reshape(-1, d)
    T = np.tile(O.csg_sdf(X if d == 3 else np.c_[X, X[:, :1]]).reshape(-1, 1), (1, n_out)).astype(np.float32)
    if sig:
        T = np.clip(T + 0.5, 0, 1)
    out = []
    for m, eng in zip(ms, ("mma.sync", "tcgen05")):
        loss = m.gradients(X, T, kind)
        assert f"dw={eng}" in m.last_kernel_variant(0), m.last_kernel_variant(0)
        out.append((loss, m.grads))
    (l0, g0), (l1, g1) = out
    t, w, b = ms[0].sizes
    assert abs(l0 - l1) <= 1e-6 * abs(l0)
    assert np.array_equal(g0[:t] != 0, g1[:t] != 0)
    assert np.linalg.norm(g0[:t] - g1[:t]) <= 1e-4 * np.linalg.norm(g0[:t])   # dY identical up to fp32 order
    for a_, r_ in ((g1[t:t + w], g0[t:t + w]), (g1[t + w:], g0[t + w:])):
        assert np.linalg.norm(a_ - r_) <= 1e-3 * np.linalg.norm(r_)


def test_train_dw_running_scale_rescales():   # the TMEM accumulators' dz scale decreasing tile by tile
    """Targets that grow along the sample order make every later tile of a
    CTA need another power-of-two dz scale than the one its accumulators
    hold, so the tcgen05 path rescales TMEM on (almost) every tile; the
    result must still match the mma.sync path's per-tile-scaled reduction."""
    from paper_2201_05989_b200 import nf
    g = _grid(nf, dims=3, levels=16, table_size=1 << 16, features=2, n_min=16, n_max=512)
    ms = []
    for eng in (SYNC, TC):
        m = nf.FieldModel(options=nf.Options(mlp_engine=eng, deterministic=True))
        m.hash_cfg = g
        m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
        m.init(5)
        ms.append(m)
    B = 1 << 17
    X = _points(B, 3, seed=11)
    ramp = np.exp2(np.linspace(-12.0, 12.0, B)).astype(np.float32).reshape(-1, 1)   # |d| spans 2^24
    T = (O.csg_sdf(X).reshape(-1, 1) * ramp).astype(np.float32)
    out = []
    for m in ms:
        loss = m.gradients(X, T, nf.LossKind.L2)
        out.append((loss, m.grads))
    (l0, g0), (l1, g1) = out
    t, w, b = ms[0].sizes
    assert abs(l0 - l1) <= 1e-6 * abs(l0)
    assert np.linalg.norm(g0[:t] - g1[:t]) <= 1e-4 * np.linalg.norm(g0[:t])
    for a_, r_ in ((g1[t:t + w], g0[t:t + w]), (g1[t + w:], g0[t + w:])):
        assert np.linalg.norm(a_ - r_) <= 1e-3 * np.linalg.norm(r_)


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("F,levels,dims", [(1, 32, 2), (4, 8, 3), (8, 4, 3)])
def test_train_dw_engines_agree_other_feature_counts(F, levels, dims, fp32):
    """The fused training kernels for F = 1, 4, 8 (no lane pairs; with fp16
    tables F = 4 takes the aliased gather staging in the tcgen05 kernel's
    canonical buffers): tcgen05 vs mma.sync dW, loss vs the oracle."""
    from paper_2201_05989_b200 import nf
    g = _grid(nf, dims=dims, levels=levels, table_size=1 << 14, features=F, n_min=4, n_max=256)
    ms = []
    for eng in (SYNC, TC):
        m = nf.FieldModel(options=nf.Options(mlp_engine=eng, table_fp32=fp32))
        m.hash_cfg = g
        m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
        m.hyper = nf.AdamHyper(lr=1e-3)
        m.init(9)
        ms.append(m)
    f = _oracle_field(ms[0], lr=1e-3, seed=9)
    B = 100000
    X = _points(B, dims, seed=13)
    T = O.csg_sdf(X if dims == 3 else np.c_[X, X[:, :1]]).reshape(-1, 1).astype(np.float32)
    out = []
    for m, eng in zip(ms, ("mma.sync", "tcgen05")):
        loss = m.gradients(X, T, nf.LossKind.Mape)
        assert f"dw={eng}" in m.last_kernel_variant(0), m.last_kernel_variant(0)
        out.append((loss, m.grads))
    (l0, g0), (l1, g1) = out
    t, w, b = ms[0].sizes
    P = ms[0].params
    if not fp32:
        P[:t] = P[:t].astype(np.float16).astype(np.float32)
    f.params[:] = P
    lo = f.train_step(X, T, O.LOSS_MAPE, 1)   # the oracle's loss on the same parameters
    assert abs(l0 - lo) <= 1e-3 * abs(lo) and abs(l1 - lo) <= 1e-3 * abs(lo), (l0, l1, lo)
    assert np.array_equal(g0[:t] != 0, g1[:t] != 0)
    assert np.linalg.norm(g0[:t] - g1[:t]) <= 1e-4 * np.linalg.norm(g0[:t])
    for a_, r_ in ((g1[t:t + w], g0[t:t + w]), (g1[t + w:], g0[t + w:])):
        assert np.linalg.norm(a_ - r_) <= 1e-3 * np.linalg.norm(r_)
