"""The sm_100a path (through the C ABI) against the committed golden vectors
(tests/golden/field_vectors.npz, written by tools/dump_golden.py from the
pinned oracle). Nothing here runs the oracle: the fixtures are the oracle.
Tolerances follow the parity contract in tests/test_gpu_parity.py."""
import hashlib

import numpy as np
import pytest

import _golden as G

pytestmark = pytest.mark.gpu


def _model(v, table_fp32=True):
    from paper_2201_05989_b200 import nf
    n_out, sig, _, seed = (int(x) for x in v["mlp"])
    m = nf.FieldModel(options=nf.Options(table_fp32=table_fp32))
    m.hash_cfg = nf.HashEncodingConfig(**G.grid_kwargs(v))
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=n_out,
                             output_activation=nf.OutputActivation.Sigmoid if sig else nf.OutputActivation.Linear)
    m.hyper = nf.AdamHyper(lr=1e-2)
    m.init(seed)
    return m


@pytest.mark.parametrize("case", G.CASES)
def test_golden_init_and_encode(case):   # model.cpp:23-37, grid.hpp:219-272
    v = G.load(case)
    m = _model(v)
    P = m.params
    assert hashlib.sha256(P.tobytes()).hexdigest() == str(v["params0_sha256"])
    Y, cache = m.encode_forward(v["X"], want_cache=True)
    assert np.array_equal(cache.rows, v["rows"])
    assert np.array_equal(cache.weights.view(np.uint32), v["weights"].view(np.uint32))
    assert np.abs(Y - v["Y"]).max() <= 1e-6 * np.abs(v["Y"]).max() + 1e-9


MATH_TOL = 1e-3   # kernel vs the exact fp16-operand emulation (tests/_fp16ref.py): fp32 summation order only


def _emulation(v):
    """The kernel's arithmetic emulated exactly on the golden inputs (fp16
    roundings of Y, weights, activations and scaled dz; fp32/f64 sums), with
    the table gradients scattered from the golden corner rows / weights. Pure
    numpy on the fixture data: no oracle call."""
    import _fp16ref as R
    n_out, sig, kind, _ = (int(x) for x in v["mlp"])
    Y = v["Y"].astype(np.float64)
    in_real = Y.shape[1]
    nW = 64 * in_real + 64 * 64 + n_out * 64
    W, b = v["mlp_params0"][:nW], v["mlp_params0"][nW:]
    shapes = [(64, in_real), (64, 64), (n_out, 64)]
    out, _, _, _ = R.forward(W, b, shapes, Y, sig)
    T = v["target"].astype(np.float64)
    n = out.size
    if kind == 0:
        dp = 2.0 * (out - T) / n
    elif kind == 1:
        dp = np.sign(out - T) / (np.abs(T) + 0.01) / n
    else:
        dp = 2.0 * (out - T) / (out * out + 0.01) / n
    _, gW, gb, dY = R.backward(W, b, shapes, Y, dp, sig, tile=64)
    L = len(v["row_offset"])
    F = in_real // L
    rows, wts = v["rows"], v["weights"]   # (L, B, corners), the golden EncodeCache
    scatter = []
    for l in range(L):
        base = (int(v["row_offset"][l]) + rows[l].astype(np.int64)) * F   # (B, corners)
        for f in range(F):
            scatter.append(((base + f).ravel(), (wts[l].astype(np.float64) * dY[:, l * F + f][:, None]).ravel()))
    return out, gW, gb, scatter


def _table_grad(scatter, size):
    g = np.zeros(size, np.float64)
    for k, c in scatter:
        np.add.at(g, k, c)
    return g


def _rel(a, r):
    return float(np.linalg.norm(np.asarray(a, np.float64) - r) / max(np.linalg.norm(np.asarray(r, np.float64)), 1e-30))


@pytest.mark.parametrize("case", G.CASES)
def test_golden_evaluate(case):   # model.cpp:102-109 (fp16 MMA operands)
    """Kernel vs emulation <= MATH_TOL * max|out| (the kernel's math); kernel vs
    the fp32 golden <= the emulation's own distance from it (the cost of fp16
    operands, computed here on the same inputs) + MATH_TOL * max|out|."""
    v = G.load(case)
    out = _model(v).evaluate(v["X"])
    ref = v["out"]
    emu = _emulation(v)[0]
    scale = np.abs(ref).max()
    assert np.abs(out - emu).max() <= MATH_TOL * scale + 1e-7
    assert np.abs(out - ref).max() <= np.abs(emu - ref).max() + MATH_TOL * scale + 1e-7


@pytest.mark.parametrize("case", G.CASES)
def test_golden_gradients(case):   # model.cpp:111-138 without the Adam step
    """Same derivation as test_gpu_headline: ||gpu - emu|| <= MATH_TOL and, by
    the triangle inequality, ||gpu - golden|| <= ||emu - golden|| + MATH_TOL
    (relative norms), per parameter group."""
    from paper_2201_05989_b200 import nf
    v = G.load(case)
    m = _model(v)
    t = m.sizes[0]
    loss = m.gradients(v["X"], v["target"], nf.LossKind(int(v["mlp"][2])))
    assert abs(loss - float(v["loss"])) <= 1e-3 * abs(float(v["loss"]))
    g = m.grads
    assert np.array_equal(np.flatnonzero(g[:t]), v["grad_table_index"])   # same touched-entry set
    _, eW, eb, egt = _emulation(v)
    e_tab = _table_grad(egt, t)[v["grad_table_index"]]
    e_mlp = np.concatenate([eW, eb])
    for a, r, e in ((g[:t][v["grad_table_index"]], v["grad_table_value"], e_tab), (g[t:], v["grad_mlp"], e_mlp)):
        assert _rel(a, e) <= MATH_TOL, (_rel(a, e), _rel(e, r))
        assert _rel(a, r) <= _rel(e, r) + MATH_TOL, (_rel(a, r), _rel(e, r))


@pytest.mark.parametrize("case", G.CASES)
def test_golden_one_train_step(case):   # model.cpp:111-138, adam.hpp:78-122 (skip-zero)
    from paper_2201_05989_b200 import nf
    v = G.load(case)
    m = _model(v)
    t = m.sizes[0]
    loss = m.train_step(v["X"], v["target"], nf.LossKind(int(v["mlp"][2])), 1)
    assert abs(loss - float(v["step1_loss"])) <= 1e-3 * abs(float(v["step1_loss"]))
    P = m.params
    idx = v["grad_table_index"]
    # untouched rows bit-identical to the oracle's (skip-zero Adam)
    assert hashlib.sha256(np.delete(P[:t], idx).tobytes()).hexdigest() == str(v["params1_untouched_sha256"])
    # touched entries and MLP parameters: Adam's first step is ±lr·sign(g) up to epsilon,
    # so they agree except where a tiny gradient flips sign (fp16 MMA operands)
    for a, r in ((P[:t][idx], v["params1_table_touched"]), (P[t:], v["params1_mlp"])):
        assert np.mean(np.abs(a - r) > 1e-5) < 0.02
