"""ctypes view of the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, by ``__graft_entry__.smoke()`` (as
the checker) and by bench.py's CPU-baseline / ``--impl reference`` legs. The
product package ``paper_2201_05989_b200`` never imports this module.

The functions below restate the reference's hot path (see nf_oracle.hpp for
the file:line citations) on numpy arrays laid out exactly like the reference's
Eigen column-major matrices: X is (B, d) C-order == d x B column-major, Y is
(B, L*F), MLP weights are (in, out) C-order == out x in column-major.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def build(native: bool = False) -> str:
    """Compile the oracle with its Makefile; returns the .so path."""
    target = "native" if native else "all"
    name = "liboracle_native.so" if native else "liboracle.so"
    subprocess.run(["make", "-s", "-C", _HERE, target], check=True)
    return os.path.join(_BUILD, name)


_LIBS = {}


def lib(native: bool = False) -> C.CDLL:
    key = bool(native)
    if key in _LIBS:
        return _LIBS[key]
    name = "liboracle_native.so" if native else "liboracle.so"
    path = os.path.join(_BUILD, name)
    if not os.path.exists(path):
        build(native)
    L = C.CDLL(path)
    _declare(L)
    _LIBS[key] = L
    return L


def _declare(L: C.CDLL) -> None:
    def d(name, res, *args):
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = list(args)

    d("orc_last_error", C.c_char_p)
    d("orc_set_threads", None, C.c_int)
    d("orc_max_threads", C.c_int)
    d("orc_growth_factor", C.c_double, _i32p)
    d("orc_levels", C.c_int64, _i32p, _u32p, _u32p, _i32p, _u64p)
    d("orc_hash", C.c_uint32, _u32p, C.c_int, C.c_uint32)
    d("orc_vertex_index", C.c_uint32, C.c_uint32, C.c_int, _u32p, C.c_int, C.c_uint32)
    d("orc_smoothstep_d", C.c_double, C.c_double)
    d("orc_weights_d", None, _f64p, C.c_int, C.c_int, _f64p)
    d("orc_weights_f", None, _f32p, C.c_int, C.c_int, _f32p)
    d("orc_voxel_f", None, C.c_float, C.c_uint32, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_float))
    for sfx, fp in (("f", _f32p), ("d", _f64p)):
        d(f"orc_encode_fwd_{sfx}", C.c_int, _i32p, fp, fp, C.c_int64, fp, _vp, _vp)
        d(f"orc_encode_bwd_{sfx}", C.c_int, _i32p, _u32p, fp, C.c_int64, fp, fp)
        d(f"orc_glorot_{sfx}", C.c_int, _i32p, C.c_uint64, fp, fp)
        d(f"orc_mlp_{sfx}", C.c_int, _i32p, fp, fp, fp, C.c_int64, fp, _vp, _vp, _vp, _vp)
        d(f"orc_loss_{sfx}", C.c_float if sfx == "f" else C.c_double, C.c_int, fp, fp, C.c_int64, fp)
    d("orc_init_tables_f", None, C.c_uint64, C.c_float, _f32p, C.c_uint64)
    d("orc_init_tables_d", None, C.c_uint64, C.c_double, _f64p, C.c_uint64)
    d("orc_psnr_f", C.c_double, _f32p, _f32p, C.c_int64)
    d("orc_adam_f", C.c_int, C.POINTER(C.c_uint64), C.c_int, _i32p, _vp, _vp, _vp, _vp, _u64p, _vp,
      _f64p, C.c_float)
    d("orc_adam_d", C.c_int, C.POINTER(C.c_uint64), C.c_int, _i32p, _vp, _vp, _vp, _vp, _u64p, _vp,
      _f64p, C.c_double)
    d("orc_lr_at", C.c_double, _i64p, C.c_int, C.c_double, C.c_double, C.c_int64)
    d("orc_default_milestones", C.c_int, C.c_int64, _i64p, C.c_int)
    d("orc_field_create", _vp, _i32p, _i32p, _f64p)
    d("orc_field_destroy", None, _vp)
    d("orc_field_init", None, _vp, C.c_uint64)
    d("orc_field_set_schedule", None, _vp, _i64p, C.c_int, C.c_double)
    d("orc_field_buffer", C.POINTER(C.c_float), _vp, C.c_int, C.POINTER(C.c_uint64))
    d("orc_field_sizes", None, _vp, _u64p)
    d("orc_field_step", C.c_uint64, _vp)
    d("orc_field_set_step", None, _vp, C.c_uint64)
    d("orc_field_train_step", C.c_int, _vp, _f32p, _f32p, C.c_int64, C.c_int, C.c_int64,
      C.POINTER(C.c_float), _vp)
    d("orc_field_evaluate", C.c_int, _vp, _f32p, C.c_int64, _f32p)
    d("orc_field_times", None, _vp, _f64p)
    d("orc_field_reset_times", None, _vp)
    d("orc_field_set_fast_mlp", None, _vp, C.c_int)
    d("orc_rng_create", _vp, C.c_uint64, C.c_uint64)
    d("orc_rng_destroy", None, _vp)
    d("orc_rng_u32", C.c_uint32, _vp)
    d("orc_rng_below", C.c_uint32, _vp, C.c_uint32)
    d("orc_rng_f32", C.c_float, _vp)
    d("orc_rng_f64", C.c_double, _vp)
    d("orc_rng_fill_f32", None, _vp, _f32p, C.c_int64)
    d("orc_rng_fill_f64", None, _vp, _f64p, C.c_int64)
    d("orc_rng_fill_u32", None, _vp, _u32p, C.c_int64)
    d("orc_image_batch", None, _vp, _f32p, C.c_int, C.c_int, C.c_int64, _f32p, _f32p)
    d("orc_make_test_image", None, C.c_int, C.c_int, _f32p)
    d("orc_csg_sdf", None, _f32p, C.c_int64, _f32p)


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    """std::invalid_argument in the reference."""


class OracleRuntimeError(OracleError, RuntimeError):
    """std::runtime_error in the reference."""


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().orc_last_error().decode()
    if status == 1:
        raise OracleInvalidArgument(msg)
    if status == 2:
        raise OracleRuntimeError(msg)
    raise OracleError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# Config mirrors (reference grid.hpp:25-57, mlp.hpp:15-40, adam.hpp:13-25)
# --------------------------------------------------------------------------
@dataclass
class GridCfg:
    levels: int = 16
    table_size: int = 1 << 14
    features: int = 2
    n_min: int = 16
    n_max: int = 512
    dims: int = 3
    smoothstep: bool = False

    def arr(self) -> np.ndarray:
        return np.array([self.levels, self.table_size, self.features, self.n_min, self.n_max,
                         self.dims, int(self.smoothstep)], dtype=np.int32)

    @property
    def output_width(self) -> int:
        return self.levels * self.features


@dataclass
class MlpCfg:
    input_width: int = 32
    hidden_layers: int = 2
    hidden_width: int = 64
    output_width: int = 3
    sigmoid: bool = False

    def arr(self) -> np.ndarray:
        return np.array([self.input_width, self.hidden_layers, self.hidden_width,
                         self.output_width, int(self.sigmoid)], dtype=np.int32)

    def layer_shapes(self) -> List[tuple]:
        shapes, fan_in = [], self.input_width
        for k in range(self.hidden_layers + 1):
            out = self.hidden_width if k < self.hidden_layers else self.output_width
            shapes.append((fan_in, out))
            fan_in = out
        return shapes

    @property
    def weight_count(self) -> int:
        return sum(i * o for i, o in self.layer_shapes())

    @property
    def bias_count(self) -> int:
        return sum(o for _, o in self.layer_shapes())


@dataclass
class Hyper:
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    l2: float = 1e-6

    def arr(self) -> np.ndarray:
        return np.array([self.lr, self.beta1, self.beta2, self.eps, self.l2], dtype=np.float64)


LOSS_L2, LOSS_MAPE, LOSS_REL_L2 = 0, 1, 2


# --------------------------------------------------------------------------
# Grid
# --------------------------------------------------------------------------
@dataclass
class LevelSpec:
    level: int
    resolution: int
    table_len: int
    dense: bool
    row_offset: int


def growth_factor(cfg: GridCfg) -> float:
    return lib().orc_growth_factor(cfg.arr())


def level_resolutions(cfg: GridCfg) -> List[LevelSpec]:
    L = max(cfg.levels, 1)
    res = np.zeros(L, np.uint32)
    ln = np.zeros(L, np.uint32)
    dn = np.zeros(L, np.int32)
    off = np.zeros(L, np.uint64)
    total = lib().orc_levels(cfg.arr(), res, ln, dn, off)
    if total < 0:
        raise OracleInvalidArgument(lib().orc_last_error().decode())
    return [LevelSpec(l, int(res[l]), int(ln[l]), bool(dn[l]), int(off[l])) for l in range(cfg.levels)]


def table_param_count(cfg: GridCfg) -> int:
    return sum(s.table_len for s in level_resolutions(cfg)) * cfg.features


def spatial_hash(coords: Sequence[int], dims: int, T: int) -> int:
    c = np.zeros(3, np.uint32)
    c[: len(coords)] = np.asarray(coords, dtype=np.uint64).astype(np.uint32)
    return int(lib().orc_hash(c, dims, T))


def grid_vertex_index(resolution: int, dense: bool, coords: Sequence[int], dims: int, T: int) -> int:
    c = np.zeros(3, np.uint32)
    c[: len(coords)] = np.asarray(coords, dtype=np.uint64).astype(np.uint32)
    return int(lib().orc_vertex_index(resolution, int(dense), c, dims, T))


def smoothstep(x: float) -> float:
    return lib().orc_smoothstep_d(x)


def interpolation_weights(frac, dims: int, smooth: bool, dtype=np.float64) -> np.ndarray:
    f = np.zeros(3, dtype)
    f[:dims] = frac
    w = np.zeros(8, dtype)
    (lib().orc_weights_d if dtype == np.float64 else lib().orc_weights_f)(f, dims, int(smooth), w)
    return w[: 1 << dims]


def voxel_of(x: float, resolution: int, half: bool):
    corner = C.c_uint32()
    frac = C.c_float()
    lib().orc_voxel_f(float(x), resolution, int(half), C.byref(corner), C.byref(frac))
    return corner.value, frac.value


def init_tables(cfg: GridCfg, seed: int, magnitude: float = 1e-4, dtype=np.float32) -> np.ndarray:
    n = table_param_count(cfg)
    p = np.zeros(n, dtype)
    if dtype == np.float32:
        lib().orc_init_tables_f(seed, magnitude, p, n)
    else:
        lib().orc_init_tables_d(seed, magnitude, p, n)
    return p


@dataclass
class EncodeCache:
    rows: np.ndarray      # (L, B, 2^d) uint32
    weights: np.ndarray   # (L, B, 2^d)


def encode_forward(cfg: GridCfg, params: np.ndarray, X: np.ndarray, want_cache: bool = True):
    dt = params.dtype
    X = np.ascontiguousarray(X, dtype=dt)
    if X.ndim != 2 or X.shape[1] != cfg.dims:
        raise OracleInvalidArgument("encode_forward: input dimensionality mismatch")
    B = X.shape[0]
    Y = np.zeros((B, cfg.output_width), dt)
    nc = 1 << cfg.dims
    rows = np.zeros((cfg.levels, B, nc), np.uint32) if want_cache else None
    wts = np.zeros((cfg.levels, B, nc), dt) if want_cache else None
    fn = lib().orc_encode_fwd_f if dt == np.float32 else lib().orc_encode_fwd_d
    _check(fn(cfg.arr(), np.ascontiguousarray(params), X, B, Y, _ptr(rows), _ptr(wts)))
    return Y, (EncodeCache(rows, wts) if want_cache else None)


def encode_backward(cfg: GridCfg, cache: EncodeCache, dY: np.ndarray, grads: np.ndarray) -> None:
    dt = grads.dtype
    dY = np.ascontiguousarray(dY, dtype=dt)
    B = dY.shape[0]
    if dY.shape[1] != cfg.output_width or cache.rows.shape[1] != B:
        raise OracleInvalidArgument("encode_backward: gradient shape does not match cache")
    fn = lib().orc_encode_bwd_f if dt == np.float32 else lib().orc_encode_bwd_d
    _check(fn(cfg.arr(), cache.rows, np.ascontiguousarray(cache.weights, dtype=dt), B, dY, grads))


# --------------------------------------------------------------------------
# MLP
# --------------------------------------------------------------------------
def glorot_init(cfg: MlpCfg, seed: int, dtype=np.float32):
    W = np.zeros(cfg.weight_count, dtype)
    b = np.zeros(cfg.bias_count, dtype)
    fn = lib().orc_glorot_f if dtype == np.float32 else lib().orc_glorot_d
    _check(fn(cfg.arr(), seed, W, b))
    return W, b


def split_weights(cfg: MlpCfg, W: np.ndarray) -> List[np.ndarray]:
    """Flat weight block -> list of (out, in) matrices (the reference's MatX)."""
    mats, off = [], 0
    for fin, fout in cfg.layer_shapes():
        mats.append(W[off: off + fin * fout].reshape(fin, fout).T)
        off += fin * fout
    return mats


def mlp_forward(cfg: MlpCfg, W, b, Y):
    dt = W.dtype
    Y = np.ascontiguousarray(Y, dtype=dt)
    if Y.shape[1] != cfg.input_width:
        raise OracleInvalidArgument("mlp_forward: input width mismatch")
    B = Y.shape[0]
    out = np.zeros((B, cfg.output_width), dt)
    fn = lib().orc_mlp_f if dt == np.float32 else lib().orc_mlp_d
    _check(fn(cfg.arr(), W, b, Y, B, out, None, None, None, None))
    return out


def mlp_forward_backward(cfg: MlpCfg, W, b, Y, dOut, gW=None, gb=None):
    """Forward then mlp_backward (grads ACCUMULATE into gW/gb, mlp.hpp:147-148)."""
    dt = W.dtype
    Y = np.ascontiguousarray(Y, dtype=dt)
    dOut = np.ascontiguousarray(dOut, dtype=dt)
    B = Y.shape[0]
    out = np.zeros((B, cfg.output_width), dt)
    gW = np.zeros_like(W) if gW is None else gW
    gb = np.zeros_like(b) if gb is None else gb
    dY = np.zeros((B, cfg.input_width), dt)
    fn = lib().orc_mlp_f if dt == np.float32 else lib().orc_mlp_d
    _check(fn(cfg.arr(), W, b, Y, B, out, _ptr(dOut), _ptr(gW), _ptr(gb), _ptr(dY)))
    return out, gW, gb, dY


# --------------------------------------------------------------------------
# Losses
# --------------------------------------------------------------------------
def loss_with_grad(kind: int, pred: np.ndarray, target: np.ndarray):
    if pred.shape != target.shape:
        raise OracleInvalidArgument("loss: shape mismatch")
    dt = pred.dtype
    p = np.ascontiguousarray(pred)
    t = np.ascontiguousarray(target, dtype=dt)
    dp = np.zeros_like(p)
    fn = lib().orc_loss_f if dt == np.float32 else lib().orc_loss_d
    return fn(kind, p, t, p.size, dp), dp


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape != b.shape:
        raise OracleInvalidArgument("psnr: shape mismatch")
    return lib().orc_psnr_f(np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32), a.size)


# --------------------------------------------------------------------------
# Adam
# --------------------------------------------------------------------------
@dataclass
class ParamGroup:
    name: str
    params: np.ndarray
    grads: np.ndarray
    apply_l2: bool = False
    skip_zero_grad: bool = False


@dataclass
class AdamState:
    step: int = 0
    m: List[np.ndarray] = field(default_factory=list)
    v: List[np.ndarray] = field(default_factory=list)

    def init(self, groups: Sequence[ParamGroup]) -> None:
        self.step = 0
        self.m = [np.zeros_like(g.params) for g in groups]
        self.v = [np.zeros_like(g.params) for g in groups]


def adam_step(state: AdamState, groups: Sequence[ParamGroup], hyper: Hyper, lr_now: float) -> None:
    ng = len(groups)
    dt = groups[0].params.dtype
    flags = np.array([[int(g.apply_l2), int(g.skip_zero_grad)] for g in groups], np.int32).ravel()
    arrp = C.c_void_p * ng
    P = arrp(*[_ptr(g.params) for g in groups])
    G = arrp(*[_ptr(g.grads) for g in groups])
    M = arrp(*[_ptr(m) for m in state.m])
    V = arrp(*[_ptr(v) for v in state.v])
    n = np.array([g.params.size for g in groups], np.uint64)
    names_b = [g.name.encode() for g in groups]
    names = (C.c_char_p * ng)(*names_b)
    st = C.c_uint64(state.step)
    fn = lib().orc_adam_f if dt == np.float32 else lib().orc_adam_d
    status = fn(C.byref(st), ng, flags, C.cast(P, C.c_void_p), C.cast(G, C.c_void_p),
                C.cast(M, C.c_void_p), C.cast(V, C.c_void_p), n, C.cast(names, C.c_void_p),
                hyper.arr(), lr_now)
    _check(status)
    state.step = int(st.value)


def lr_at(milestones: Sequence[int], factor: float, base_lr: float, step: int) -> float:
    ms = np.asarray(milestones, np.int64)
    return lib().orc_lr_at(np.ascontiguousarray(ms), len(ms), factor, base_lr, step)


def default_milestones(total_steps: int) -> List[int]:
    out = np.zeros(64, np.int64)
    n = lib().orc_default_milestones(total_steps, out, 64)
    return [int(x) for x in out[:n]]


# --------------------------------------------------------------------------
# Field model (FieldModel, model.hpp:21-63)
# --------------------------------------------------------------------------
class Field:
    def __init__(self, grid: GridCfg, mlp: MlpCfg, hyper: Hyper = Hyper(), native: bool = False):
        self._lib = lib(native)
        mlp = MlpCfg(grid.output_width, mlp.hidden_layers, mlp.hidden_width, mlp.output_width, mlp.sigmoid)
        self.grid, self.mlp, self.hyper = grid, mlp, hyper
        self.h = self._lib.orc_field_create(grid.arr(), mlp.arr(), hyper.arr())
        if not self.h:
            raise OracleInvalidArgument(self._lib.orc_last_error().decode())
        sz = np.zeros(3, np.uint64)
        self._lib.orc_field_sizes(self.h, sz)
        self.n_tab, self.n_w, self.n_b = (int(x) for x in sz)

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.orc_field_destroy(self.h)
            self.h = None

    def init(self, seed: int) -> None:
        self._lib.orc_field_init(self.h, seed)

    def set_schedule(self, milestones: Sequence[int], factor: float = 0.33) -> None:
        ms = np.ascontiguousarray(np.asarray(milestones, np.int64))
        self._lib.orc_field_set_schedule(self.h, ms, len(ms), factor)

    def buffer(self, which: int) -> np.ndarray:
        n = C.c_uint64()
        p = self._lib.orc_field_buffer(self.h, which, C.byref(n))
        return np.ctypeslib.as_array(p, shape=(n.value,))

    params = property(lambda self: self.buffer(0))
    grads = property(lambda self: self.buffer(1))
    m = property(lambda self: self.buffer(2))
    v = property(lambda self: self.buffer(3))

    @property
    def step(self) -> int:
        return int(self._lib.orc_field_step(self.h))

    @step.setter
    def step(self, s: int) -> None:
        self._lib.orc_field_set_step(self.h, s)

    def train_step(self, X, target, loss_kind: int, step: int, want_pred: bool = False):
        X = np.ascontiguousarray(X, np.float32)
        target = np.ascontiguousarray(target, np.float32)
        B = X.shape[0]
        loss = C.c_float()
        pred = np.zeros((B, self.mlp.output_width), np.float32) if want_pred else None
        status = self._lib.orc_field_train_step(self.h, X, target, B, loss_kind, step, C.byref(loss), _ptr(pred))
        if status:
            msg = self._lib.orc_last_error().decode()
            raise (OracleInvalidArgument if status == 1 else OracleRuntimeError)(msg)
        return (loss.value, pred) if want_pred else loss.value

    def evaluate(self, X) -> np.ndarray:
        X = np.ascontiguousarray(X, np.float32)
        out = np.zeros((X.shape[0], self.mlp.output_width), np.float32)
        status = self._lib.orc_field_evaluate(self.h, X, X.shape[0], out)
        if status:
            raise OracleInvalidArgument(self._lib.orc_last_error().decode())
        return out

    def phase_times(self) -> dict:
        t = np.zeros(6, np.float64)
        self._lib.orc_field_times(self.h, t)
        keys = ("encode_fwd", "mlp_fwd", "loss", "mlp_bwd", "encode_bwd", "adam")
        return dict(zip(keys, (float(x) for x in t)))

    def reset_times(self) -> None:
        self._lib.orc_field_reset_times(self.h)

    def set_fast_mlp(self, on: bool = True) -> None:
        """CPU-baseline timing only: the MLP through cache-blocked FMA GEMMs
        standing in for the reference's Eigen GEMMs (nf_oracle.hpp fast::)."""
        self._lib.orc_field_set_fast_mlp(self.h, int(on))


# --------------------------------------------------------------------------
# Checkpoint (io.cpp:222-351): NFC1 | HGE1 | MLP1 | ADM1, little-endian
# --------------------------------------------------------------------------
def save_checkpoint(field: "Field", path: str, n_frequencies: int = 10) -> None:   # io.cpp:222-285
    import struct
    g, m = field.grid, field.mlp
    P, M, V = field.params, field.m, field.v
    out = bytearray(b"NFC1" + struct.pack("<II", 0, n_frequencies) + b"HGE1")
    out += struct.pack("<7I", g.dims, g.levels, g.table_size, g.features, g.n_min, g.n_max, int(g.smoothstep))
    for lv in level_resolutions(g):                      # io.cpp:241-244
        off = lv.row_offset * g.features
        out += struct.pack("<Q", lv.table_len) + P[off:off + lv.table_len * g.features].astype("<f4").tobytes()
    out += b"MLP1" + struct.pack("<5I", m.input_width, m.hidden_layers, m.hidden_width, m.output_width,
                                 int(m.sigmoid))
    wo, bo = field.n_tab, field.n_tab + field.n_w
    for (i, o) in m.layer_shapes():                      # io.cpp:264-267: W_k then b_k
        out += P[wo:wo + o * i].astype("<f4").tobytes() + P[bo:bo + o].astype("<f4").tobytes()
        wo += o * i
        bo += o
    out += b"ADM1" + struct.pack("<QI", field.step, 3)
    off = 0
    for n in (field.n_tab, field.n_w, field.n_b):        # io.cpp:273-277
        out += struct.pack("<Q", n) + M[off:off + n].astype("<f4").tobytes() + V[off:off + n].astype("<f4").tobytes()
        off += n
    with open(path, "wb") as f:
        f.write(bytes(out))


def load_checkpoint(path: str, hyper: "Hyper" = None) -> "Field":   # io.cpp:287-351
    import struct
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise OracleRuntimeError("cannot read checkpoint: " + path) from None
    pos = 0

    def take(n, what="truncated file"):
        nonlocal pos
        if pos + n > len(data):
            raise OracleRuntimeError("checkpoint: " + what)
        b = data[pos:pos + n]
        pos += n
        return b

    def tag(t, what):
        if pos + 4 > len(data) or data[pos:pos + 4] != t:
            raise OracleRuntimeError(f"checkpoint: missing {what} section")
        take(4)

    def floats(n):
        return np.frombuffer(take(4 * n, "truncated float block"), "<f4").astype(np.float32)

    tag(b"NFC1", "file header")
    encoder, _ = struct.unpack("<II", take(8))
    if encoder != 0:
        raise OracleRuntimeError("checkpoint: only the hash encoder is restated")
    tag(b"HGE1", "feature table")
    d, L, T, F, nmin, nmax, interp = struct.unpack("<7I", take(28))
    g = GridCfg(levels=L, table_size=T, features=F, n_min=nmin, n_max=nmax, dims=d, smoothstep=bool(interp))
    tab = []
    for lv in level_resolutions(g):
        (n,) = struct.unpack("<Q", take(8))
        if n != lv.table_len:
            raise OracleRuntimeError("checkpoint: level length mismatch")
        tab.append(floats(n * F))
    tag(b"MLP1", "MLP parameters")
    iw, hl, hw, ow, act = struct.unpack("<5I", take(20))
    f = Field(g, MlpCfg(hidden_layers=hl, hidden_width=hw, output_width=ow, sigmoid=bool(act)), hyper or Hyper())
    Ws, bs = [], []
    for (i, o) in f.mlp.layer_shapes():
        Ws.append(floats(o * i))
        bs.append(floats(o))
    tag(b"ADM1", "optimizer state")
    step, ng = struct.unpack("<QI", take(12))
    ms, vs = [], []
    for _ in range(ng):
        (n,) = struct.unpack("<Q", take(8))
        ms.append(floats(n))
        vs.append(floats(n))
    f.params[:] = np.concatenate(tab + Ws + bs)
    f.m[:] = np.concatenate(ms)
    f.v[:] = np.concatenate(vs)
    f.step = step
    return f


# --------------------------------------------------------------------------
# Inference consumers (tasks.cpp:195-356), vectorised over rays / points; the
# field is any function (n, d) float32 -> n values (FieldFn, tasks.hpp:70).
# --------------------------------------------------------------------------
def _cross(a, b):   # Eigen cross
    return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]])


def _normalized(v):   # v / sqrt(squaredNorm)
    return v / np.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])


def render_sdf_shaded(field, position, target, up, fov_deg, W, H):   # tasks.cpp:233-329
    import math
    pos = np.asarray(position, np.float64)
    fwd = _normalized(np.asarray(target, np.float64) - pos)
    right = _normalized(_cross(fwd, np.asarray(up, np.float64)))
    up2 = _cross(right, fwd)
    half_tan = math.tan(0.5 * fov_deg * math.pi / 180.0)
    aspect = float(W) / float(H)
    i = np.arange(W * H)
    x, y = (i % W).astype(np.float64), (i // W).astype(np.float64)
    u = ((2.0 * (x + 0.5)) / W - 1.0) * half_tan * aspect
    v = (1.0 - (2.0 * (y + 0.5)) / H) * half_tan
    d = [(fwd[k] + u * right[k]) + v * up2[k] for k in range(3)]
    nn = np.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
    d = np.stack([dk / nn for dk in d], axis=1)
    t0 = np.zeros(W * H)
    t1 = np.full(W * H, np.inf)
    fail = np.zeros(W * H, bool)
    with np.errstate(divide="ignore", invalid="ignore"):
        for k in range(3):   # ray_unit_cube (tasks.cpp:213-229)
            inv = 1.0 / d[:, k]
            near, far = (0.0 - pos[k]) * inv, (1.0 - pos[k]) * inv
            sw = near > far
            near, far = np.where(sw, far, near), np.where(sw, near, far)
            t0 = np.where(t0 < near, near, t0)
            t1 = np.where(far < t1, far, t1)
            fail |= t0 > t1
    act = np.nonzero(~fail)[0]
    t, texit = t0[act] + 1e-6, t1[act]
    rgb = np.ones((W * H, 3), np.float32)
    hit_pix, hit_t = [], []
    for _ in range(256):
        if act.size == 0:
            break
        pts = np.clip(pos[None, :] + t[:, None] * d[act], 0.0, 1.0).astype(np.float32)
        val = np.asarray(field(pts), np.float32).reshape(-1).astype(np.float64)
        hit = val < 1e-4
        hit_pix.append(act[hit])
        hit_t.append(t[hit])
        t2 = t + val
        keep = ~hit & (t2 <= texit)
        act, t, texit = act[keep], t2[keep], texit[keep]
    if hit_pix:
        hp, ht = np.concatenate(hit_pix), np.concatenate(hit_t)
        if hp.size:
            p = pos[None, :] + ht[:, None] * d[hp]
            probes = np.repeat(p[:, None, :], 6, axis=1)
            for a in range(3):
                probes[:, 2 * a, a] += 1e-3
                probes[:, 2 * a + 1, a] -= 1e-3
            vals = np.asarray(field(np.clip(probes.reshape(-1, 3), 0.0, 1.0).astype(np.float32)),
                              np.float32).reshape(-1, 6)
            n = np.stack([(vals[:, 2 * a] - vals[:, 2 * a + 1]).astype(np.float64) for a in range(3)], axis=1)
            ln = np.sqrt((n[:, 0] * n[:, 0] + n[:, 1] * n[:, 1]) + n[:, 2] * n[:, 2])
            with np.errstate(divide="ignore", invalid="ignore"):
                n = np.where(ln[:, None] > 0, n / ln[:, None], n)
            dd = d[hp]
            dot = (n[:, 0] * -dd[:, 0] + n[:, 1] * -dd[:, 1]) + n[:, 2] * -dd[:, 2]
            shade = (0.15 + 0.85 * np.where(dot > 0, dot, 0.0)).astype(np.float32)
            rgb[hp] = (np.float32(0.9) * shade)[:, None]
    return rgb


def iou(field, oracle_sign, n_points, rng: "Pcg32", lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):   # tasks.cpp:331-356
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    both = either = 0
    for done in range(0, n_points, 1 << 16):
        n = min(1 << 16, n_points - done)
        P = lo[None, :] + (hi - lo)[None, :] * rng.doubles(3 * n).reshape(n, 3)
        pred = np.asarray(field(P.astype(np.float32)), np.float32).reshape(-1)
        m_in = pred < 0
        o_in = np.array([oracle_sign(P[i]) < 0 for i in range(n)])
        both += int(np.sum(m_in & o_in))
        either += int(np.sum(m_in | o_in))
    return 1.0 if either == 0 else both / either


# --------------------------------------------------------------------------
# NeRF. PARITY UNPINNED: the reference has no NeRF
# (SPEC.md:8); these functions restate the paper's Appendix E
# and §5.4 and are the checker for
# paper_2201_05989_b200/csrc/nerf.cu. fp32 scalar arithmetic in the device
# kernel's order (no contraction) for the marching, float64 for compositing.
# --------------------------------------------------------------------------
NERF_RES = 128
NERF_DT = np.float32(1.7320508075688772) / np.float32(1024.0)


def _spread3(v):
    v &= 0x7F
    v = (v | (v << 8)) & 0x0000F00F
    v = (v | (v << 4)) & 0x000C30C3
    v = (v | (v << 2)) & 0x00249249
    return v


def morton3(x, y, z):
    return _spread3(x) | (_spread3(y) << 1) | (_spread3(z) << 2)


def nerf_march(rays, bits, max_steps=1024):   # PAPER.md:904-936 (fixed step, occupancy skip)
    """Samples of a ray = the grid points t_k = t_base + k dt (t_base = t0 + dt/2,
    t_k < t1) whose occupancy cell is set, in k order, capped at max_steps.
    Empty points jump floor(tn / dt) - 1 points (>= 1) towards the next cell
    boundary, which never skips a point past it (so any split of the k range,
    e.g. the kernel's 32 lanes per ray, yields the same set)."""
    f = np.float32
    rays = np.asarray(rays, np.float32)
    bits = np.asarray(bits, np.uint8)
    counts, out = [], []

    def cell(p):
        c = int(p * f(NERF_RES))
        return min(max(c, 0), NERF_RES - 1)

    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        for r in rays:
            o, d = r[:3], r[3:]
            t0, t1 = f(-np.inf), f(np.inf)
            for k in range(3):
                inv = f(1.0) / d[k]
                a, b = (f(0.0) - o[k]) * inv, (f(1.0) - o[k]) * inv
                t0 = np.fmax(t0, np.fmin(a, b))
                t1 = np.fmin(t1, np.fmax(a, b))
            t0 = np.fmax(t0, f(0.0))
            n = 0
            if t1 > t0:
                tb = t0 + f(0.5) * NERF_DT
                kmax = int(np.ceil((t1 - tb) / NERF_DT)) + 1
                k = 0
                while k < kmax:
                    t = tb + f(k) * NERF_DT
                    if not t < t1:
                        break
                    p = [o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]]
                    c = [cell(v) for v in p]
                    m = morton3(c[0], c[1], c[2])
                    if (bits[m >> 3] >> (m & 7)) & 1:
                        if n < max_steps:
                            out.append(p)
                        n += 1
                        k += 1
                        continue
                    tn = f(np.inf)
                    for a_ in range(3):
                        cb = f(c[a_] + (1 if d[a_] > 0 else 0))
                        ta = (cb / f(NERF_RES) - p[a_]) / d[a_]
                        tn = np.fmin(tn, ta)
                    steps = np.floor(tn / NERF_DT) - f(1.0)
                    k += (int(steps) if steps < 1e6 else 1000000) if steps > 1 else 1
            counts.append(min(n, max_steps))
    return np.array(counts, np.uint32), np.array(out, np.float32).reshape(-1, 3)


def nerf_composite(counts, raw, rgb, target, bg=(1.0, 1.0, 1.0), dt=float(NERF_DT)):
    """Volume rendering C = sum T_i a_i c_i + T_end bg, a = 1 - exp(-exp(raw) dt),
    transmittance stop at 1e-4; L2 loss averaged over rays x 3 and its gradients
    w.r.t. the per-sample colours and log-densities (float64)."""
    raw = np.asarray(raw, np.float64)
    rgb = np.asarray(rgb, np.float64)
    target = np.asarray(target, np.float64)
    bg = np.asarray(bg, np.float64)
    R = len(counts)
    color = np.zeros((R, 3))
    d_rgb = np.zeros_like(rgb)
    d_raw = np.zeros_like(raw)
    loss = 0.0
    off = 0
    for r, n in enumerate(counts):
        T, C, used, ws = 1.0, np.zeros(3), 0, []
        for i in range(off, off + int(n)):
            if T < 1e-4:
                break
            a = 1.0 - np.exp(-np.exp(raw[i]) * dt)
            ws.append(T * a)
            C += T * a * rgb[i]
            T *= 1.0 - a
            used += 1
        color[r] = C + T * bg
        e = color[r] - target[r]
        loss += float(e @ e)
        g = 2.0 * e / (3.0 * R)
        P = np.zeros(3)
        T2 = 1.0
        for j in range(used):
            i = off + j
            a = 1.0 - np.exp(-np.exp(raw[i]) * dt)
            P += ws[j] * rgb[i]
            T2 *= 1.0 - a
            d_rgb[i] = ws[j] * g
            d_raw[i] = dt * ((T2 * rgb[i] - (C - P) - T * bg) @ g) * np.exp(min(raw[i], 15.0))
        off += int(n)
    return color, d_rgb, d_raw, loss


def sh4(d):   # real spherical harmonics up to degree 4 (16 coefficients)
    x, y, z = d[:, 0].astype(np.float64), d[:, 1].astype(np.float64), d[:, 2].astype(np.float64)
    xy, xz, yz, x2, y2, z2 = x * y, x * z, y * z, x * x, y * y, z * z
    return np.stack([
        np.full_like(x, 0.28209479177387814), -0.48860251190291987 * y, 0.48860251190291987 * z,
        -0.48860251190291987 * x, 1.0925484305920792 * xy, -1.0925484305920792 * yz,
        0.94617469575755997 * z2 - 0.31539156525251999, -1.0925484305920792 * xz,
        0.54627421529603959 * x2 - 0.54627421529603959 * y2, 0.59004358992664352 * y * (-3.0 * x2 + y2),
        2.8906114426405538 * xy * z, 0.45704579946446572 * y * (1.0 - 5.0 * z2),
        0.3731763325901154 * z * (5.0 * z2 - 3.0), 0.45704579946446572 * x * (1.0 - 5.0 * z2),
        1.4453057213202769 * z * (x2 - y2), 0.59004358992664352 * x * (-x2 + 3.0 * y2)], axis=1)


NERF_SCENE = [((0.40, 0.45, 0.50), 0.18, (0.90, 0.30, 0.20)), ((0.62, 0.55, 0.45), 0.14, (0.20, 0.70, 0.90)),
              ((0.50, 0.30, 0.62), 0.10, (0.85, 0.85, 0.25))]


def nerf_scene(P):   # the synthetic procedural scene: (sigma (n,), rgb (n, 3))
    P = np.asarray(P, np.float64)
    sig = np.zeros(len(P))
    best = np.full(len(P), 1e9)
    col = np.zeros((len(P), 3))
    for c, r, rgb in NERF_SCENE:
        dist = np.linalg.norm(P - np.array(c), axis=1) - r
        with np.errstate(over="ignore"):
            sig += 80.0 / (1.0 + np.exp(dist * 150.0))
        m = dist < best
        best = np.where(m, dist, best)
        col[m] = rgb
    tex = 0.65 + 0.35 * np.sin(18.0 * (P[:, 0] + 0.7 * P[:, 1] - 0.4 * P[:, 2]))
    return sig, col * tex[:, None]


def nerf_pixel_rays(cam, w, h, focal):
    cam = np.asarray(cam, np.float64)
    i = np.arange(w * h)
    x, y = i % w, i // w
    u = (x + 0.5 - 0.5 * w) / focal
    v = (0.5 * h - y - 0.5) / focal
    d = cam[3:6][None, :] + u[:, None] * cam[6:9][None, :] + v[:, None] * cam[9:12][None, :]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.repeat(cam[None, :3], w * h, axis=0), d


def nerf_scene_render(cam, w, h, focal, bg=(1.0, 1.0, 1.0)):   # fine marching of the analytic scene (float64)
    o, d = nerf_pixel_rays(cam, w, h, focal)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        a, b = (0.0 - o) * inv, (1.0 - o) * inv
        t0 = np.fmax(np.nanmax(np.fmin(a, b), axis=1), 0.0)
        t1 = np.nanmin(np.fmax(a, b), axis=1)
    dt = float(NERF_DT)
    T = np.ones(len(o))
    C = np.zeros((len(o), 3))
    t = t0 + 0.5 * dt
    live = t1 > t0
    while live.any():
        live &= (t < t1) & (T >= 1e-4)
        if not live.any():
            break
        s, c = nerf_scene(o[live] + t[live, None] * d[live])
        a = 1.0 - np.exp(-s * dt)
        C[live] += (T[live] * a)[:, None] * c
        T[live] *= 1.0 - a
        t = t + dt
    return C + T[:, None] * np.asarray(bg)


# --------------------------------------------------------------------------
# RNG and fixtures
# --------------------------------------------------------------------------
class Pcg32:
    def __init__(self, seed: int, seq: int = 1):
        self._lib = lib()
        self.h = self._lib.orc_rng_create(seed, seq)

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.orc_rng_destroy(self.h)
            self.h = None

    def next_u32(self) -> int:
        return int(self._lib.orc_rng_u32(self.h))

    def next_below(self, bound: int) -> int:
        return int(self._lib.orc_rng_below(self.h, bound))

    def next_float(self) -> float:
        return float(self._lib.orc_rng_f32(self.h))

    def next_double(self) -> float:
        return float(self._lib.orc_rng_f64(self.h))

    def floats(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.float32)
        self._lib.orc_rng_fill_f32(self.h, out, n)
        return out

    def doubles(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.float64)
        self._lib.orc_rng_fill_f64(self.h, out, n)
        return out

    def u32s(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint32)
        self._lib.orc_rng_fill_u32(self.h, out, n)
        return out

    def image_batch(self, rgb: np.ndarray, w: int, h: int, B: int):
        X = np.zeros((B, 2), np.float32)
        t = np.zeros((B, 3), np.float32)
        self._lib.orc_image_batch(self.h, np.ascontiguousarray(rgb, np.float32), w, h, B, X, t)
        return X, t


def make_test_image(w: int, h: int) -> np.ndarray:
    """(w*h, 3) float32, pixel i = y*w + x (reference tests/helpers.hpp:99-125)."""
    rgb = np.zeros((w * h, 3), np.float32)
    lib().orc_make_test_image(w, h, rgb)
    return rgb


def csg_sdf(X: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float32)
    out = np.zeros(X.shape[0], np.float32)
    lib().orc_csg_sdf(X, X.shape[0], out)
    return out


def set_threads(n: int) -> None:
    lib().orc_set_threads(n)
