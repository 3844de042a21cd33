"""World-size-2 data-parallel checks on CPU (gloo), SURVEY.md §8e.

The GPU path all-reduces the fp32 gradient slab with NCCL inside the library;
these tests prove the host-side contract it relies on, with the oracle as the
per-rank compute engine and gloo as the collective:
  * shard() covers the global batch exactly once;
  * rank gradients normalised by the GLOBAL count sum to the single-process
    gradient of the whole batch (losses.hpp:16 normalises by pred.size());
  * the replicated Adam step after the all-reduce leaves both ranks with
    bit-identical parameters that move like the single-process step
    (skip-zero sees the global gradient);
  * the 128-byte communicator id broadcast reaches every rank unchanged.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2201_05989_b200.dp import broadcast_unique_id, grad_scale, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_partitions_batch():
    for B in (0, 1, 7, 1000, 1 << 18):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                s, e = shard(B, r, world)
                cover.extend(range(s, e))
                assert abs((e - s) - B / world) < 1
            assert cover == list(range(B))
    with pytest.raises(ValueError):
        shard(10, 2, 2)


GCFG = O.GridCfg(levels=8, table_size=1 << 10, features=2, n_min=4, n_max=64, dims=3)
MCFG = O.MlpCfg(input_width=16, hidden_layers=2, hidden_width=16, output_width=1)


def _grads(t, W, b, X, T, kind):
    """Oracle gradient of the loss over (X, T), locally normalised (losses.hpp)."""
    Y, cache = O.encode_forward(GCFG, t, X)
    pred = O.mlp_forward(MCFG, W, b, Y)
    loss, dp = O.loss_with_grad(kind, pred, T)
    _, gW, gb, dY = O.mlp_forward_backward(MCFG, W, b, Y, dp)
    gt = np.zeros_like(t)
    O.encode_backward(GCFG, cache, dY, gt)
    return loss, np.concatenate([gt, gW, gb])


def _problem(B=333):
    t = O.init_tables(GCFG, 7, 1e-2, np.float64)
    W, b = O.glorot_init(MCFG, 8, np.float64)
    rng = O.Pcg32(9, 1)
    X = rng.doubles(B * 3).reshape(B, 3)
    T = O.csg_sdf(X.astype(np.float32)).astype(np.float64).reshape(B, 1)
    return t, W, b, X, T


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, W, b, X, T = _problem()
        B = X.shape[0]
        s, e = shard(B, rank, world)
        loss_l, g = _grads(t, W, b, X[s:e], T[s:e], O.LOSS_MAPE)
        g = g * grad_scale(e - s, B)                  # == normalising by the global count
        gt = torch.from_numpy(g)
        dist.all_reduce(gt)                           # the library does this with NCCL
        lt = torch.tensor([loss_l * (e - s) / B], dtype=torch.float64)
        dist.all_reduce(lt)
        # replicated Adam on the reduced gradient (float32, as on the GPU)
        n_t, n_w = t.size, W.size
        P = np.concatenate([t, W, b]).astype(np.float32)
        G = gt.numpy().astype(np.float32)
        groups = [O.ParamGroup("tables", P[:n_t], G[:n_t], False, True),
                  O.ParamGroup("mlp_weights", P[n_t:n_t + n_w], G[n_t:n_t + n_w], True, False),
                  O.ParamGroup("mlp_biases", P[n_t + n_w:], G[n_t + n_w:], False, False)]
        st = O.AdamState()
        st.init(groups)
        O.adam_step(st, groups, O.Hyper(lr=1e-3), np.float32(1e-3))
        uid = broadcast_unique_id(lambda: bytes(range(128)), rank)
        q.put((rank, gt.numpy(), float(lt.item()), P, uid))
    finally:
        dist.destroy_process_group()


def test_two_rank_gradient_allreduce_equals_full_batch():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t, W, b, X, T = _problem()
    loss_full, g_full = _grads(t, W, b, X, T, O.LOSS_MAPE)
    for rank, g, loss, P, uid in res:
        np.testing.assert_allclose(g, g_full, rtol=1e-10, atol=1e-14)
        assert abs(loss - loss_full) <= 1e-12 * abs(loss_full)
        assert uid == bytes(range(128))
    assert np.array_equal(res[0][3], res[1][3])        # replicas stay identical after Adam
    # ...and equal to the single-process step on the full batch
    n_t, n_w = t.size, W.size
    P = np.concatenate([t, W, b]).astype(np.float32)
    G = g_full.astype(np.float32)
    groups = [O.ParamGroup("tables", P[:n_t], G[:n_t], False, True),
              O.ParamGroup("mlp_weights", P[n_t:n_t + n_w], G[n_t:n_t + n_w], True, False),
              O.ParamGroup("mlp_biases", P[n_t + n_w:], G[n_t + n_w:], False, False)]
    st = O.AdamState()
    st.init(groups)
    O.adam_step(st, groups, O.Hyper(lr=1e-3), np.float32(1e-3))
    # gradients agree to ~1e-16 relative (float64 sums in a different order); after the
    # float32 cast Adam moves each parameter by ~lr*sign(g): compare signs of the updates
    d_dp, d_sp = res[0][3] - np.concatenate([t, W, b]).astype(np.float32), P - np.concatenate([t, W, b]).astype(np.float32)
    big = np.abs(G) > 1e-9 * np.abs(G).max()
    assert np.array_equal(np.sign(d_dp[big]), np.sign(d_sp[big]))
