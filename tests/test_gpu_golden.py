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


@pytest.mark.parametrize("case", G.CASES)
def test_golden_evaluate(case):   # model.cpp:102-109 (fp16 MMA operands)
    v = G.load(case)
    out = _model(v).evaluate(v["X"])
    ref = v["out"]
    assert np.abs(out - ref).max() <= 1e-2 * np.abs(ref).max() + 1e-4


@pytest.mark.parametrize("case", G.CASES)
def test_golden_gradients(case):   # model.cpp:111-138 without the Adam step
    from paper_2201_05989_b200 import nf
    v = G.load(case)
    m = _model(v)
    t = m.sizes[0]
    loss = m.gradients(v["X"], v["target"], nf.LossKind(int(v["mlp"][2])))
    assert abs(loss - float(v["loss"])) <= 1e-3 * abs(float(v["loss"]))
    g = m.grads
    assert np.array_equal(np.flatnonzero(g[:t]), v["grad_table_index"])   # same touched-entry set
    for a, r in ((g[:t][v["grad_table_index"]], v["grad_table_value"]), (g[t:], v["grad_mlp"])):
        assert np.linalg.norm(a - r) <= 6e-2 * np.linalg.norm(r)


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
