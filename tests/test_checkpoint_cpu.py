"""Checkpoint format (io.cpp:222-351) and train report CSV (io.cpp:189-220):
oracle restatement round trips and the reference's corrupt-file cases
(test_tasks.cpp:255-337), CPU only."""
import os

import numpy as np
import pytest

import oracle as O


def _field(seed=9):
    f = O.Field(O.GridCfg(levels=3, table_size=1 << 8, features=2, n_min=4, n_max=16, dims=2),
                O.MlpCfg(hidden_layers=2, hidden_width=64, output_width=3, sigmoid=True), O.Hyper(lr=1e-2))
    f.init(seed)
    rng = O.Pcg32(seed, 1)
    for step in range(1, 6):
        X = rng.floats(64 * 2).reshape(64, 2)
        f.train_step(X, np.full((64, 3), 0.5, np.float32), 0, step)
    return f


def test_oracle_checkpoint_round_trip_bit_exact(tmp_path):   # test_tasks.cpp:284-324
    f = _field()
    p = str(tmp_path / "ck.bin")
    O.save_checkpoint(f, p)
    g = O.load_checkpoint(p, O.Hyper(lr=1e-2))
    for a, b in ((f.params, g.params), (f.m, g.m), (f.v, g.v)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert g.step == f.step == 5
    X = O.Pcg32(2, 0).floats(64).reshape(32, 2)
    assert np.array_equal(f.evaluate(X), g.evaluate(X))
    T = np.full((32, 3), 0.5, np.float32)
    assert f.train_step(X, T, 0, 21) == g.train_step(X, T, 0, 21)
    assert np.array_equal(f.params, g.params)
    # re-saving the loaded model reproduces the file byte for byte
    q = str(tmp_path / "ck2.bin")
    O.save_checkpoint(O.load_checkpoint(p), q)
    assert open(p, "rb").read() == open(q, "rb").read()


def test_oracle_checkpoint_layout(tmp_path):   # io.cpp:226-277 section order and sizes
    f = _field()
    p = str(tmp_path / "ck.bin")
    O.save_checkpoint(f, p)
    data = open(p, "rb").read()
    assert data[:4] == b"NFC1" and data[12:16] == b"HGE1"
    n = f.n_tab + f.n_w + f.n_b
    # header 12 + HGE1 4+28 + 3 level lengths + MLP1 4+20 + ADM1 4+8+4 + 3 group lengths, then floats
    assert len(data) == 12 + 32 + 3 * 8 + 24 + 16 + 3 * 8 + 4 * (n + 2 * n)


@pytest.mark.parametrize("content,msg", [(b"not a checkpoint", "missing file header"),
                                          (b"NFC1\0\0\0\0\n\0\0\0HGE1\2\0", "truncated")])
def test_oracle_checkpoint_rejects_corrupt(tmp_path, content, msg):   # test_tasks.cpp:326-337
    p = str(tmp_path / "bad.bin")
    open(p, "wb").write(content)
    with pytest.raises(O.OracleRuntimeError, match=msg):
        O.load_checkpoint(p)
    with pytest.raises(O.OracleRuntimeError, match="cannot read checkpoint"):
        O.load_checkpoint(str(tmp_path / "nonexistent_checkpoint.bin"))


def test_report_csv_round_trip(tmp_path):   # test_tasks.cpp:255-281
    from paper_2201_05989_b200 import nf
    rep = nf.TrainReport([nf.TrainReportRow(s, 0.25 * s, 1.0 / (s + 3), 20.0 + s / 7.0, 1e-2 * 0.33 ** s)
                          for s in range(5)])
    p = str(tmp_path / "report.csv")
    nf.write_report_csv(rep, p)
    assert open(p).readline().strip() == "step,time_s,loss,metric,lr"
    back = nf.read_report_csv(p)
    assert len(back.rows) == 5
    for a, b in zip(rep.rows, back.rows):
        assert a.step == b.step
        for k in ("time_s", "loss", "metric", "lr"):
            assert getattr(b, k) == pytest.approx(getattr(a, k), rel=1e-9)
