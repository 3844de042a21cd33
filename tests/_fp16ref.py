"""numpy emulation of the GPU MLP's storage precision (test-side checker).

Restates mlp.hpp:104-158 in float64 but rounds to fp16 exactly where the
sm_100a kernel stores fp16 operands: the layer inputs (Y and every hidden
activation), the weights, and the backward dz operands. Bias gradients use
the unrounded dz (the kernel sums its fp32 C fragments). Agreement with this
emulation (tight tolerance) proves the kernel's math; agreement with the fp32
oracle (loose tolerance) measures the precision choice.
"""
import numpy as np


def h(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def split(W, b, shapes):
    mats, biases, wo, bo = [], [], 0, 0
    for out, fin in shapes:
        mats.append(np.asarray(W[wo: wo + out * fin], np.float64).reshape(fin, out).T)
        biases.append(np.asarray(b[bo: bo + out], np.float64))
        wo += out * fin
        bo += out
    return mats, biases


def forward(W, b, shapes, Y, sigmoid):
    mats, biases = split(W, b, shapes)
    a = h(Y)
    acts, masks = [a], []
    for k, (Wk, bk) in enumerate(zip(mats, biases)):
        z = a @ h(Wk).T + bk
        if k + 1 < len(mats):
            m = z > 0
            masks.append(m)
            a = h(np.where(m, z, 0.0))
            acts.append(a)
        else:
            out = 1 / (1 + np.exp(-z)) if sigmoid else z
    return out, acts, masks, mats


def tile_scale(d, tile=64):
    """The kernel's per-tile power-of-two scale: max|d| * s < 16 over each
    64-sample k_train tile (TS = 16 x 4 warps, field_kernels.cuh)."""
    s = np.ones((d.shape[0], 1))
    for r in range(0, d.shape[0], tile):
        mx = np.abs(d[r:r + tile]).max()
        if mx > 0:
            _, ex = np.frexp(np.float32(mx))
            s[r:r + tile] = 2.0 ** max(-100, min(100, 4 - int(ex)))
    return s


def backward(W, b, shapes, Y, dOut, sigmoid, tile=64):
    out, acts, masks, mats = forward(W, b, shapes, Y, sigmoid)
    dz = np.asarray(dOut, np.float64)
    if sigmoid:
        dz = dz * (out * (1 - out))
    sc = tile_scale(dz, tile)
    gW, gb = [None] * len(mats), [None] * len(mats)
    for k in range(len(mats) - 1, -1, -1):
        dzh = h(dz * sc) / sc
        gb[k] = dzh.sum(0)   # the kernel forms db on the tensor cores from the fp16 dz
        gW[k] = dzh.T @ acts[k]
        da = dzh @ h(mats[k])
        if k > 0:
            dz = np.where(masks[k - 1], da, 0.0)
        else:
            dY = da
    flatW = np.concatenate([g.T.ravel() for g in gW])
    return out, flatW, np.concatenate(gb), dY


def touched_set_unexplained(got, ref, emu, floor=1e-4):
    """Table entries whose touched status (gradient != 0) differs between the
    kernel and the fp32 oracle, and that the fp16 operands do not explain.

    A touched entry's oracle gradient can be exactly zero (a sample with every
    ReLU unit off in fp32 gives dY = 0) while the fp16-operand step gives a
    value at the noise floor (seen: 1.6e-10 on the GPU, 2.1e-10 in the
    emulation, 0 in the oracle). Such an entry is explained when the emulation
    sits on the kernel's side, or when both gradients are below
    floor * max|ref|. Returns (all differing indices, unexplained indices)."""
    got, ref, emu = (np.asarray(v) for v in (got, ref, emu))
    d = np.flatnonzero((got != 0) != (ref != 0))
    same_side = (emu[d] != 0) == (got[d] != 0)
    tiny = np.maximum(np.abs(got[d]), np.abs(ref[d])) <= floor * np.abs(ref).max()
    return d, d[~(same_side | tiny)]
