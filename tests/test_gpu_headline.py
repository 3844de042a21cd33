"""Parity of the EXACT kernel instantiation bench.py measures.

bench.py runs the default ``Options()``: fp16 shadow tables, the fused
``k_train`` with its corner staging aliased into the activation/dz rows
(``stage_alias=1``, field_kernels.cuh StageAlias), lane-pair gathers and
reductions. Every test here asserts (through ``nfg_last_kernel_variant``) that
this is the instantiation that ran, then compares it with the CPU oracle on
identical inputs and parameters (model.cpp:111-138).

Tolerances and where they come from:
  * the oracle runs on the fp16-ROUNDED tables (the values the kernel gathers);
    its Adam updates the fp32 master, as the kernel's does;
  * loss: <= 1e-3 relative (contract);
  * touched table entries: identical set (contract), up to entries whose
    fp32 gradient is exactly zero while the fp16-operand step leaves a value
    at the noise floor (reproduced by the emulation; _fp16ref.touched_set_unexplained);
  * gradients are checked twice. (1) Against ``tests/_fp16ref.py``, an exact
    numpy emulation of the kernel's fp16 operand roundings (Y, activations,
    weights, dz): <= 1e-3 in norm — this checks the kernel's math.
    (2) Against the fp32 oracle: by the triangle inequality
    ||gpu - oracle|| <= ||gpu - emu|| + ||emu - oracle||, so the bound is
    the emulation's own distance from the oracle (the cost of fp16 operands,
    measured on the same batch on the CPU, not asserted) + 1e-3. On a TRAINED
    field that distance is < 1e-2 and the §8c contract (1e-2) is asserted
    directly. At init (tables ~1e-4, pre-activations near zero) fp16 rounding
    flips ReLU masks of near-zero units, and the emulation itself sits ~3%
    from the oracle (DESIGN.md §3 "Precision").
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

CFG2 = dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)   # BASELINE config 2
CFG1 = dict(dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=1024)   # BASELINE config 1

# (grid, n_out, sigmoid, loss kind, lr, full batch)
# smoothstep interpolation (grid.hpp:112-133) through the same default
# options: fp16 tables, the interp=smooth encoding instantiation
CFGS = dict(dims=3, levels=16, table_size=1 << 16, features=2, n_min=16, n_max=512, interpolation=1)
CASES = {
    "config2": (CFG2, 1, False, 1, 1e-4, 1 << 18),
    "config1": (CFG1, 3, True, 0, 1e-2, 1 << 16),
    "smooth3d": (CFGS, 1, False, 1, 1e-2, 1 << 15),
}
MATH_TOL = 1e-3      # gpu vs the fp16-operand emulation (kernel math; measured <= 4.2e-4)
# smoothstep fields: 30 trained runs (tools/headline_margins.py smooth3d)
# measured median 2e-6 / 2e-4 (two batches) and max 3.5e-3 for the table
# gradients: a sample near a ReLU boundary can flip between the kernel and
# the emulation when the smoothstep-weighted Y rounds differently in fp16.
# A wrong interpolation instantiation is off by O(1).
MATH_TOL_SMOOTH = 1e-2
# Well-trained smoothstep fields also show rare rows whose gradient is exactly
# zero in the kernel but not in the oracle (or the reverse): about 1 in 40
# batches, at most 8 entries of ~1e5 touched, each below 2e-3 of the largest
# gradient. Diagnosed (profiles/headline_margins_smooth3d_diag_r2.log): the
# row is touched by a single sample whose kernel prediction equals its target
# exactly, so the MAPE gradient sign(0) / den is 0, while the fp32 oracle's
# prediction is one rounding away. The build before this round's kernel
# changes shows the same (profiles/headline_margins_smooth3d_r2_old_new.log).
SMOOTH_ODD_ENTRIES, SMOOTH_ODD_FLOOR = 16, 1e-2
CONTRACT = 1e-2      # SURVEY.md §8c table/MLP gradient contract (trained fields)


def _nf():
    from paper_2201_05989_b200 import nf
    return nf


def _model(case):
    nf = _nf()
    grid, n_out, sig, _, lr, _ = CASES[case]
    m = nf.FieldModel()   # default Options(): exactly what bench.py runs
    assert m.options == nf.Options()
    m.hash_cfg = nf.HashEncodingConfig(**grid)
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=n_out,
                             output_activation=nf.OutputActivation.Sigmoid if sig else nf.OutputActivation.Linear)
    m.hyper = nf.AdamHyper(lr=lr)
    m.init(1337)
    return m


def _ocfg(grid):
    return O.GridCfg(levels=grid["levels"], table_size=grid["table_size"], features=grid["features"],
                     n_min=grid["n_min"], n_max=grid["n_max"], dims=grid["dims"],
                     smoothstep=bool(grid.get("interpolation", 0)))


def _batch(case, B, seed):
    grid, n_out, sig, _, _, _ = CASES[case]
    rng = O.Pcg32(seed, 2)
    X = rng.floats(B * grid["dims"]).reshape(B, grid["dims"])
    if grid["dims"] == 3:
        T = O.csg_sdf(X).reshape(B, 1)
    else:   # the procedural test image (helpers.hpp:99-125) at the sample positions
        w = 1024
        rgb = O.make_test_image(w, w)
        ix = np.minimum((X * w).astype(np.int64), w - 1)
        T = np.ascontiguousarray(rgb[ix[:, 1] * w + ix[:, 0]], np.float32)
    return X, T


def _assert_headline_variant(m):
    v = m.last_kernel_variant(0)
    d = m.hash_cfg.dims
    smooth = int(m.hash_cfg.interpolation) == 1
    assert v.startswith("k_train src=0 grad=0 sink=0") and f"d={d} " in v, v
    assert "F=2 table=f16 in_steps=2 hidden=2 stage_alias=1" in v, v
    assert "dw=tcgen05" in v, v   # the default engine bench.py measures (profiles/tc_train_r2.md)
    assert ("interp=smooth" if smooth else "interp=linear") in v, v   # interpolation fixed at compile time


def _train_gpu(m, case, steps, seed=99):
    """Move the field off its ~1e-4 init with the headline kernel itself."""
    kind = CASES[case][3]
    for s in range(1, steps + 1):
        X, T = _batch(case, 1 << 14, seed + s)
        m.train_step(X, T, kind, s)


def _oracle_grads(case, P, sizes, X, T):
    """The reference's composition (model.cpp:111-138) on fp16-rounded tables,
    plus the fp16-operand emulation of the same step (tests/_fp16ref.py)."""
    import _fp16ref as R
    grid, n_out, sig, kind, _, _ = CASES[case]
    og = _ocfg(grid)
    t, w, _ = sizes
    tab16 = P[:t].astype(np.float16).astype(np.float32)
    W, b = P[t:t + w], P[t + w:]
    mc = O.MlpCfg(grid["levels"] * grid["features"], 2, 64, n_out, sig)
    Y, cache = O.encode_forward(og, tab16, X)
    pred = O.mlp_forward(mc, W, b, Y)
    loss, dp = O.loss_with_grad(kind, pred, T)
    _, gW, gb, dY = O.mlp_forward_backward(mc, W, b, Y, dp)
    gt = np.zeros(t, np.float32)
    O.encode_backward(og, cache, dY, gt)
    shapes = [(64, mc.input_width), (64, 64), (n_out, 64)]
    out_e, _, _, _ = R.forward(W, b, shapes, Y, sig)
    _, dpe = O.loss_with_grad(kind, out_e.astype(np.float32), T)
    _, eW, eb, eY = R.backward(W, b, shapes, Y, dpe, sig, tile=64)
    ge = np.zeros(t, np.float32)
    O.encode_backward(og, cache, eY.astype(np.float32), ge)
    ref = (gt, gW, gb)
    emu = (ge, eW.astype(np.float32), eb.astype(np.float32))
    return loss, ref, emu, cache


def _rel(a, r):
    return float(np.linalg.norm(np.asarray(a, np.float64) - r) / max(np.linalg.norm(np.asarray(r, np.float64)), 1e-30))


# smooth3d runs on trained fields only (lr 1e-2, as config 1): at init, and
# after 20 steps at lr 1e-3, its smoothstep-weighted features sit near 1e-5,
# in fp16's subnormal range, where the kernel's and the oracle's differently
# ordered blends round Y apart and the emulation is no longer exact
# (measured up to 5e-3 from the kernel)
@pytest.mark.parametrize("ragged", [False, True])
@pytest.mark.parametrize("case,state", [("config2", "init"), ("config2", "trained"), ("config1", "init"),
                                        ("config1", "trained"), ("smooth3d", "trained")])
def test_headline_gradients(case, ragged, state):   # model.cpp:111-138 via the benchmarked k_train
    m = _model(case)
    if state == "trained":
        _train_gpu(m, case, 20)
    full = CASES[case][5]
    B = full - 37 if ragged else full   # ragged: a partial last 64-sample tile
    X, T = _batch(case, B, seed=5 + ragged)
    P = m.params
    assert (m.grads == 0).all()
    lg = m.gradients(X, T, CASES[case][3])
    _assert_headline_variant(m)
    G = m.grads
    lo, ref, emu, _ = _oracle_grads(case, P, m.sizes, X, T)
    t, w, _ = m.sizes
    got = (G[:t], G[t:t + w], G[t + w:])
    assert abs(lg - lo) <= 1e-3 * abs(lo), (lg, lo)
    # identical touched-entry set, up to entries at the fp16-operand noise floor
    # (tests/_fp16ref.py::touched_set_unexplained; at most 1e-5 of the touched set)
    import _fp16ref as R
    smooth = case == "smooth3d"
    diff_set, bad = R.touched_set_unexplained(got[0], ref[0], emu[0], floor=SMOOTH_ODD_FLOOR if smooth else 1e-4)
    if smooth:
        assert diff_set.size <= SMOOTH_ODD_ENTRIES, diff_set.size
    assert bad.size == 0, ("touched-entry sets differ", bad[:10], got[0][bad[:10]], ref[0][bad[:10]], emu[0][bad[:10]])
    assert diff_set.size <= 1e-5 * np.count_nonzero(ref[0]) + 1, diff_set.size
    report = {}
    for name, a, r, e in zip(("tables", "mlp_weights", "mlp_biases"), got, ref, emu):
        d_emu, d_ref, emu_ref = _rel(a, e), _rel(a, r), _rel(e, r)
        report[name] = (d_emu, d_ref, emu_ref)
        assert d_emu <= (MATH_TOL_SMOOTH if case == "smooth3d" else MATH_TOL), (name, report)
        assert d_ref <= emu_ref + MATH_TOL, (name, report)
        if state == "trained" and case != "smooth3d":   # §8c's contract is quoted on configs 1 and 2
            assert d_ref <= CONTRACT, (name, report)
        big = np.abs(r) > 1e-2 * np.abs(r).max()
        agree = float(np.mean(np.sign(a[big]) == np.sign(r[big])))
        assert agree > 0.99, (name, agree, report)
    print(case, B, state, report)


def _oracle_step(case, m, P, Mo, Vo, step, X, T):
    """One reference train_step from the GPU field's exact state: gradients on
    the fp16-rounded tables, Adam (adam.hpp:78-122) on the fp32 master."""
    grid, n_out, sig, kind, lr, _ = CASES[case]
    t, w, _ = m.sizes
    loss, (gt, gW, gb), _, cache = _oracle_grads(case, P, m.sizes, X, T)
    p = P.copy()
    mm, vv = Mo.copy(), Vo.copy()
    g = np.concatenate([gt, gW, gb]).astype(np.float32)
    groups = [O.ParamGroup("tables", p[:t], g[:t], False, True),
              O.ParamGroup("mlp_weights", p[t:t + w], g[t:t + w], True, False),
              O.ParamGroup("mlp_biases", p[t + w:], g[t + w:], False, False)]
    st = O.AdamState(step=step - 1, m=[mm[:t], mm[t:t + w], mm[t + w:]], v=[vv[:t], vv[t:t + w], vv[t + w:]])
    g_before = g.copy()   # adam_step zeroes the gradients (adam.hpp:118-120)
    O.adam_step(st, groups, O.Hyper(lr=lr), np.float32(lr))
    return loss, p, g_before, cache


def _step_checks(case, m, before, after, ref_p, ref_g, cache, lg, lo):
    grid, _, _, _, lr, _ = CASES[case]
    t = m.sizes[0]
    F = grid["features"]
    assert abs(lg - lo) <= 1e-3 * abs(lo), (lg, lo)
    # skip-zero: entries with a zero oracle gradient are bit-identical to before
    untouched = ref_g[:t] == 0
    moved = np.flatnonzero(after[:t][untouched].view(np.uint32) != before[:t][untouched].view(np.uint32))
    assert moved.size <= (SMOOTH_ODD_ENTRIES if case == "smooth3d" else 0), moved.size
    # every touched row changed
    specs = O.level_resolutions(_ocfg(grid))
    touched = np.zeros(t // F, bool)
    for l in range(grid["levels"]):
        touched[specs[l].row_offset + cache.rows[l].ravel().astype(np.int64)] = True
    changed = np.any((after[:t] != before[:t]).reshape(-1, F), axis=1)
    assert not changed[~touched].any()
    # one-step parameters: Adam moves each entry by <= ~lr; the fp16 operand
    # choice perturbs the step only where a gradient is tiny against sqrt(v)
    d = np.abs(after - ref_p)
    assert np.quantile(d, 0.99) <= 0.05 * lr, np.quantile(d, [0.5, 0.99, 1.0])
    assert d.max() <= 2.5 * lr, d.max()


@pytest.mark.parametrize("path", ["plain", "streamed", "device"])
@pytest.mark.parametrize("ragged", [False, True])
@pytest.mark.parametrize("case", ["config2", "config1", "smooth3d"])
def test_headline_train_step(case, ragged, path):   # model.cpp:111-138 + adam.hpp:78-122, one step
    """One full step through each public entry: numpy arrays (staged copies),
    pinned host pointers (B >= 2^15: chunked H2D streamed under the running
    kernel) and device pointers (the bench loop), from a trained state whose
    parameters and Adam moments the oracle copies exactly."""
    import torch
    nf = _nf()
    m = _model(case)
    kind = CASES[case][3]
    _train_gpu(m, case, 10)   # also warms the field up (streaming starts after one plain step)
    full = CASES[case][5]
    B = full - 37 if ragged else full
    X, T = _batch(case, B, seed=31 + ragged)
    step, Mo, Vo = m.adam_state()
    before = m.params
    lo, ref_p, ref_g, cache = _oracle_step(case, m, before, Mo, Vo, step + 1, X, T)
    if path == "plain":
        lg = m.train_step(X, T, kind, step + 1)
    elif path == "streamed":
        Xh, Th = nf.PinnedBuffer(X.shape), nf.PinnedBuffer(T.shape)
        try:
            Xh.array[:] = X
            Th.array[:] = T
            lg = m.train_step_host_ptr(Xh.ptr, Th.ptr, B, kind, step + 1)
        finally:
            Xh.free()
            Th.free()
    else:
        Xd = torch.from_numpy(X).cuda()
        Td = torch.from_numpy(T).cuda()
        loss_d = torch.zeros(1, device="cuda")
        m.train_step_device(Xd, Td, B, B, kind, step + 1, loss_out=loss_d)
        m.check()
        lg = float(loss_d.item())
    _assert_headline_variant(m)
    assert m.step == step + 1
    after = m.params
    _step_checks(case, m, before, after, ref_p, ref_g, cache, lg, lo)
    assert (m.grads == 0).all()   # adam.hpp:118-120


def test_headline_streamed_invalid_last_chunk_untouched():   # grid.hpp:226-229 on the benchmarked variant
    nf = _nf()
    from paper_2201_05989_b200._lib import NfgInvalidArgument
    m = _model("config2")
    _train_gpu(m, "config2", 3)
    B = 1 << 18
    X, T = _batch("config2", B, seed=77)
    Xh, Th = nf.PinnedBuffer(X.shape), nf.PinnedBuffer(T.shape)
    try:
        Xh.array[:] = X
        Th.array[:] = T
        Xh.array[B - 3, 1] = np.nan
        step, m0, v0 = m.adam_state()
        before = m.params
        with pytest.raises(NfgInvalidArgument, match="non-finite"):
            m.train_step_host_ptr(Xh.ptr, Th.ptr, B, 1, step + 1)
        _assert_headline_variant(m)
        s1, m1, v1 = m.adam_state()
        assert s1 == step and np.array_equal(m.params, before) and (m.grads == 0).all()
        assert np.array_equal(m0, m1) and np.array_equal(v0, v1)
    finally:
        Xh.free()
        Th.free()
