"""Checkpoint interop on the GPU path (io.cpp:222-351; test_tasks.cpp:284-337):
files written by the sm_100a library are byte-identical to the oracle's
restatement of save_checkpoint for the same state, oracle files load into the
device model bit-exactly, and a deterministic-mode resume takes identical steps."""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import _nf

pytestmark = pytest.mark.gpu


def _image_model(nf, det=False, seed=9):
    m = nf.FieldModel(options=nf.Options(deterministic=det))
    m.hash_cfg = nf.HashEncodingConfig(levels=3, table_size=1 << 8, features=2, n_min=4, n_max=16, dims=2)
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=3,
                             output_activation=nf.OutputActivation.Sigmoid)
    m.hyper = nf.AdamHyper(lr=1e-2)
    m.init(seed)
    rng = O.Pcg32(seed, 1)
    for step in range(1, 21):
        X = rng.floats(64 * 2).reshape(64, 2)
        m.train_step(X, np.full((64, 3), 0.5, np.float32), nf.LossKind.L2, step)
    return m


def test_gpu_file_is_byte_identical_to_reference_format(tmp_path):
    nf = _nf()
    m = _image_model(nf)
    p = str(tmp_path / "gpu.bin")
    nf.save_checkpoint(m, p)
    # the oracle holding the same state writes the same bytes
    f = O.Field(O.GridCfg(levels=3, table_size=1 << 8, features=2, n_min=4, n_max=16, dims=2),
                O.MlpCfg(hidden_layers=2, hidden_width=64, output_width=3, sigmoid=True), O.Hyper(lr=1e-2))
    f.init(0)
    step, mm, vv = m.adam_state()
    f.params[:] = m.params
    f.m[:] = mm
    f.v[:] = vv
    f.step = step
    q = str(tmp_path / "oracle.bin")
    O.save_checkpoint(f, q)
    assert open(p, "rb").read() == open(q, "rb").read()
    # and the oracle reads the GPU file back exactly
    g = O.load_checkpoint(p)
    assert np.array_equal(g.params, m.params) and g.step == 20


def test_oracle_file_loads_bit_exactly(tmp_path):
    nf = _nf()
    f = O.Field(O.GridCfg(levels=16, table_size=1 << 12, features=2, n_min=16, n_max=512, dims=3),
                O.MlpCfg(hidden_layers=2, hidden_width=64, output_width=1), O.Hyper(lr=1e-3))
    f.init(4)
    rng = O.Pcg32(4, 2)
    for step in range(1, 4):
        X = rng.floats(512 * 3).reshape(512, 3)
        f.train_step(X, O.csg_sdf(X).reshape(-1, 1), O.LOSS_MAPE, step)
    p = str(tmp_path / "o.bin")
    O.save_checkpoint(f, p)
    m = nf.FieldModel()
    m.hyper = nf.AdamHyper(lr=1e-3)
    nf.load_checkpoint(m, p)
    assert m.hash_cfg.dims == 3 and m.hash_cfg.table_size == 1 << 12 and m.mlp_cfg.output_width == 1
    step, mm, vv = m.adam_state()
    assert step == 3
    for a, b in ((m.params, f.params), (mm, f.m), (vv, f.v)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    X = rng.floats(256 * 3).reshape(256, 3)
    out, ref = m.evaluate(X), f.evaluate(X)
    assert np.abs(out - ref).max() <= 5e-3 * np.abs(ref).max() + 1e-5


def test_round_trip_and_resume_bit_exact(tmp_path):   # test_tasks.cpp:284-324
    nf = _nf()
    a = _image_model(nf, det=True)
    p = str(tmp_path / "ck.bin")
    nf.save_checkpoint(a, p)
    b = nf.FieldModel(options=nf.Options(deterministic=True))
    nf.load_checkpoint(b, p)
    X = O.Pcg32(2, 0).floats(64).reshape(32, 2)
    assert np.abs(a.evaluate(X) - b.evaluate(X)).max() == 0.0
    assert b.adam_state()[0] == a.adam_state()[0]
    b.hyper = a.hyper
    b.schedule = a.schedule
    T = np.full((32, 3), 0.5, np.float32)
    l1 = a.train_step(X, T, nf.LossKind.L2, 21)
    l2 = b.train_step(X, T, nf.LossKind.L2, 21)
    assert l1 == l2
    assert np.abs(a.evaluate(X) - b.evaluate(X)).max() == 0.0
    assert np.array_equal(a.params.view(np.uint32), b.params.view(np.uint32))


def test_rejects_corrupt_files(tmp_path):   # test_tasks.cpp:326-337
    nf = _nf()
    from paper_2201_05989_b200 import _lib as L
    p = str(tmp_path / "bad.bin")
    open(p, "wb").write(b"not a checkpoint")
    m = nf.FieldModel()
    with pytest.raises(L.NfgIOError, match="missing file header"):
        nf.load_checkpoint(m, p)
    with pytest.raises(L.NfgIOError, match="cannot read checkpoint"):
        nf.load_checkpoint(m, str(tmp_path / "nonexistent_checkpoint.bin"))
    good = _image_model(nf)
    nf.save_checkpoint(good, p)
    data = open(p, "rb").read()
    open(p, "wb").write(data[: len(data) // 2])
    with pytest.raises(L.NfgIOError, match="truncated"):
        nf.load_checkpoint(m, p)
