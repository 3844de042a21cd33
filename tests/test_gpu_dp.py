"""Data-parallel path on one GPU through a 1-rank NCCL communicator: the
chunked all-reduce on the comm stream + per-chunk Adam (and the scratch
reduction) must take exactly the steps of the single-process path
(deterministic mode: bit-identical parameters), and abort the same way."""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import _nf

pytestmark = pytest.mark.gpu


def _pair(nf, det, exchange=0, table_fp32=False):
    import torch  # noqa: F401  (loads torch's libnccl for the communicator)
    plain = nf.Context(0)
    dp = nf.Context(0)
    dp.attach_comm(nf.Context.unique_id(), 0, 1)
    models = []
    for ctx in (plain, dp):
        m = nf.FieldModel(ctx, options=nf.Options(deterministic=det, dp_exchange=exchange, table_fp32=table_fp32))
        m.hash_cfg = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)
        m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
        m.hyper = nf.AdamHyper(lr=1e-3)
        m.init(11)
        models.append(m)
    return models, (plain, dp)


def test_chunked_allreduce_adam_matches_single_process():
    nf = _nf()
    (a, b), ctxs = _pair(nf, det=True)
    rng = O.Pcg32(3, 3)
    for step in range(1, 4):
        X = rng.floats(20000 * 3).reshape(-1, 3)
        T = O.csg_sdf(X).reshape(-1, 1)
        la = a.train_step(X, T, nf.LossKind.Mape, step)
        lb = b.train_step(X, T, nf.LossKind.Mape, step)
        assert la == lb
    assert a.adam_state()[0] == b.adam_state()[0] == 3
    for x, y in ((a.params, b.params), (a.adam_state()[1], b.adam_state()[1]), (a.adam_state()[2], b.adam_state()[2])):
        assert np.array_equal(np.asarray(x).view(np.uint32), np.asarray(y).view(np.uint32))
    assert not b.grads.any()   # Adam zeroed every gradient chunk


def test_dp_fused_path_and_invalid_input():
    nf = _nf()
    (a, b), ctxs = _pair(nf, det=False)
    rng = O.Pcg32(4, 4)
    X = rng.floats(3 * (1 << 16)).reshape(-1, 3)
    T = O.csg_sdf(X).reshape(-1, 1)
    la = a.train_step(X, T, nf.LossKind.Mape, 1)
    lb = b.train_step(X, T, nf.LossKind.Mape, 1)
    assert abs(la - lb) <= 1e-5 * abs(la)
    d = np.abs(a.params - b.params)
    assert np.mean(d > 1e-6) < 0.01
    before = b.params
    bad = X.copy()
    bad[7, 1] = 1.5
    with pytest.raises(ValueError):
        b.train_step(bad, T, nf.LossKind.Mape, 2)
    assert np.array_equal(b.params, before) and b.adam_state()[0] == 1 and not b.grads.any()
    lb2 = b.train_step(X, T, nf.LossKind.Mape, 2)
    assert np.isfinite(lb2)


@pytest.mark.parametrize("exchange", [1, 2])
def test_dp_streamed_host_pointer_steps(exchange):
    """Pinned host buffers with B >= 2^15 through the data-parallel path: the
    fused kernel waits for streamed chunks while the scratch reduction,
    exchange and Adam are queued behind it; train_step returns once the
    reduced loss / flags are known (after the last scatter of the level-
    pipelined exchange, which reads the staged inputs), and the next step's
    copies overwrite the staging buffers under the previous Adam. Losses and
    parameters track the single-process streamed path."""
    nf = _nf()
    (a, b), ctxs = _pair(nf, det=False, exchange=exchange)
    B = 1 << 16
    bufs = [(nf.PinnedBuffer((B, 3)), nf.PinnedBuffer((B, 1))) for _ in range(2)]
    try:
        rng = O.Pcg32(5, 5)
        for step in range(1, 6):   # step 1 warms both fields up, steps 2-5 stream
            X = rng.floats(3 * B).reshape(-1, 3)
            T = O.csg_sdf(X).reshape(-1, 1)
            losses = []
            for m, (xh, th) in zip((a, b), bufs):
                xh.array[:] = X
                th.array[:] = T
                losses.append(m.train_step_host_ptr(xh.ptr, th.ptr, B, nf.LossKind.Mape, step))
            assert abs(losses[0] - losses[1]) <= 1e-4 * abs(losses[0]), (step, losses)
        assert a.step == b.step == 5
        d = np.abs(a.params - b.params)
        assert np.mean(d > 1e-5) < 0.03
        assert not b.grads.any()
    finally:
        for xh, th in bufs:
            xh.free()
            th.free()


def test_broadcast_and_comm_info():
    """nfg_field_broadcast on a 1-rank communicator keeps the state (root is
    itself) and refreshes the fp16 shadow; comm_info reports NCCL's own view;
    DataParallelTrainer broadcasts at construction."""
    nf = _nf()
    from paper_2201_05989_b200.dp import DataParallelTrainer
    (a, b), (plain, dp) = _pair(nf, det=False)
    assert plain.comm_info() == (0, 1) and dp.comm_info() == (0, 1)
    rng = O.Pcg32(6, 6)
    X = rng.floats(3 * 4096).reshape(-1, 3)
    T = O.csg_sdf(X).reshape(-1, 1)
    b.train_step(X, T, nf.LossKind.Mape, 1)
    p0, (s0, m0, v0) = b.params, b.adam_state()
    b.broadcast(0)
    p1, (s1, m1, v1) = b.params, b.adam_state()
    assert s0 == s1 == 1
    for x, y in ((p0, p1), (m0, m1), (v0, v1)):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    out0 = b.evaluate(X[:256])
    DataParallelTrainer(b, 0, 1)   # world 1: attach is a no-op, broadcast still runs
    assert np.array_equal(b.evaluate(X[:256]), out0)
    with pytest.raises(ValueError):
        b.broadcast(1)   # root outside the communicator


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("exchange", [1, 2])   # NFG_DP_ALLREDUCE, NFG_DP_LEVELS
def test_dp_exchanges_track_single_process(exchange, fp32):
    """Both data-parallel exchanges on a 1-rank communicator against the
    single-process fused step. NFG_DP_LEVELS runs the fused kernel with dY
    stored, scatters the table gradients level group by level group (finest
    first) and all-reduces / updates each group separately: every gradient
    range must be reduced and updated exactly once (all gradients zero after
    Adam, every level moves), and the steps track the fused single-process path
    (same loss to fp32 summation order; scatter order differs)."""
    nf = _nf()
    (a, b), ctxs = _pair(nf, det=False, exchange=exchange, table_fp32=fp32)
    rng = O.Pcg32(7, 7)
    P0 = b.params
    for step in range(1, 4):
        X = rng.floats(3 * 50000).reshape(-1, 3)
        T = O.csg_sdf(X).reshape(-1, 1)
        la = a.train_step(X, T, nf.LossKind.Mape, step)
        lb = b.train_step(X, T, nf.LossKind.Mape, step)
        assert abs(la - lb) <= 1e-5 * abs(la), (step, la, lb)
        assert not b.grads.any()
        if exchange == 2:
            assert "sink=1" in b.last_kernel_variant(0), b.last_kernel_variant(0)   # dY stored, not scattered
        else:
            assert "sink=0" in b.last_kernel_variant(0), b.last_kernel_variant(0)
    assert a.step == b.step == 3
    d = np.abs(a.params - b.params)
    assert np.mean(d > 1e-5) < 0.02
    # every level group (and the MLP) was updated
    moved = b.params != P0
    t = b.sizes[0]
    g = O.GridCfg(levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, dims=3)
    for sp in O.level_resolutions(g):
        lo, hi = 2 * sp.row_offset, 2 * (sp.row_offset + sp.table_len)
        assert moved[lo:hi].any(), sp
    assert moved[t:].mean() > 0.9


def test_dp_levels_nonfinite_stands_down():   # adam.hpp:86-90 through the level-pipelined exchange
    nf = _nf()
    from paper_2201_05989_b200._lib import NfgNonFinite
    (a, b), ctxs = _pair(nf, det=False, exchange=2)
    rng = O.Pcg32(8, 8)
    X = rng.floats(3 * 40000).reshape(-1, 3)
    T = O.csg_sdf(X).reshape(-1, 1)
    b.train_step(X, T, nf.LossKind.Mape, 1)
    before = b.params
    T2 = T.copy()
    T2[123, 0] = np.nan
    with pytest.raises(NfgNonFinite):
        b.train_step(X, T2, nf.LossKind.L2, 2)
    assert np.array_equal(b.params.view(np.uint32), before.view(np.uint32))
    assert b.step == 1
    assert np.isfinite(b.train_step(X, T, nf.LossKind.Mape, 2))
