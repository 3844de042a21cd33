"""Python mirror of the reference's hot-path API (namespace ``nf``), backed by
the sm_100a library through the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/nf/{grid,mlp,adam,losses,model}.hpp:

* ``HashEncodingConfig``, ``MlpConfig``, ``AdamHyper``, ``LrSchedule`` — the
  reference's config structs (grid.hpp:25-57, mlp.hpp:15-40, adam.hpp:13-25,124-137).
* ``FieldModel`` — model.hpp:21-63. Set ``hash_cfg`` / ``mlp_cfg`` / ``hyper`` /
  ``schedule`` then call ``init(seed)``; ``train_step`` and ``evaluate`` run on
  the GPU. Public members of the reference (``tables``, ``mlp``, Adam state)
  are exposed as host mirrors that read/write device memory.
* Matrices are numpy arrays shaped (B, rows): C-order (B, d) is exactly the
  reference's column-major d x B ``MatX``.

Errors: ``ValueError`` (std::invalid_argument), ``NfgNonFinite``
(std::runtime_error from adam_step), ``NfgUnsupported`` (valid for the
reference but not built for sm_100a, e.g. hidden_width > 64).
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


class Interpolation(enum.IntEnum):   # grid.hpp:20
    Linear = 0
    Smoothstep = 1


class OutputActivation(enum.IntEnum):   # mlp.hpp:13
    Linear = 0
    Sigmoid = 1


class LossKind(enum.IntEnum):   # model.hpp:17
    L2 = 0
    Mape = 1
    RelativeL2 = 2


@dataclass
class HashEncodingConfig:   # grid.hpp:25-57
    levels: int = 16
    table_size: int = 1 << 14
    features: int = 2
    n_min: int = 16
    n_max: int = 512
    dims: int = 3
    interpolation: Interpolation = Interpolation.Linear

    def c(self) -> L.nfg_grid_config:
        return L.nfg_grid_config(self.levels, self.table_size, self.features, self.n_min, self.n_max, self.dims,
                                 int(self.interpolation))

    def validate(self) -> None:
        level_resolutions(self)

    def growth_factor(self) -> float:
        return L.load().nfg_growth_factor(C.byref(self.c()))

    def output_width(self) -> int:
        return self.levels * self.features


@dataclass
class GridLevelSpec:   # grid.hpp:59-64
    level: int
    resolution: int
    table_len: int
    dense: bool
    row_offset: int


def level_resolutions(cfg: HashEncodingConfig) -> List[GridLevelSpec]:   # grid.hpp:66-84
    lib = L.load()
    n = max(int(cfg.levels), 1)
    arr = (L.nfg_level_spec * n)()
    got = lib.nfg_level_resolutions(C.byref(cfg.c()), arr, n)
    if got < 0:
        raise L.NfgInvalidArgument(L.NFG_EINVAL, lib.nfg_last_error().decode())
    return [GridLevelSpec(a.level, a.resolution, a.table_len, bool(a.dense), a.row_offset) for a in arr[:got]]


def spatial_hash(coords: Sequence[int], dims: int, table_size: int) -> int:   # grid.hpp:88-95
    c = (C.c_uint32 * 3)(*([int(x) & 0xFFFFFFFF for x in coords] + [0] * (3 - len(coords))))
    return int(L.load().nfg_spatial_hash(c, dims, table_size))


def grid_vertex_index(spec: GridLevelSpec, coords: Sequence[int], dims: int, table_size: int) -> int:
    """grid.hpp:100-110: row-major (first coordinate fastest, stride N+1) at dense
    levels, the spatial hash otherwise."""
    if spec.dense:
        idx, stride = 0, 1
        for i in range(dims):
            idx += int(coords[i]) * stride
            stride *= spec.resolution + 1
        return idx & 0xFFFFFFFF
    return spatial_hash(coords, dims, table_size)


def psnr(a, b) -> float:   # losses.hpp:63-71 (host metric)
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise L.NfgInvalidArgument(L.NFG_EINVAL, "psnr: shape mismatch")
    mse = float(((a - b) ** 2).sum() / a.size) if a.size else 0.0
    return 100.0 if mse <= 0 else min(100.0, -10.0 * np.log10(mse))


def set_threads(n: int) -> None:   # tasks.cpp:17-25
    """The reference caps OpenMP/Eigen threads (1 = deterministic mode). On the
    GPU path the equivalent switch is Options(deterministic=True); this is a
    no-op kept for API parity."""
    del n


@dataclass
class MlpConfig:   # mlp.hpp:15-40
    input_width: int = 32
    hidden_layers: int = 2
    hidden_width: int = 64
    output_width: int = 3
    output_activation: OutputActivation = OutputActivation.Linear

    def c(self) -> L.nfg_mlp_config:
        return L.nfg_mlp_config(self.input_width, self.hidden_layers, self.hidden_width, self.output_width,
                                int(self.output_activation))

    def layer_count(self) -> int:
        return self.hidden_layers + 1

    def layer_shapes(self):
        shapes, fin = [], self.input_width
        for k in range(self.layer_count()):
            out = self.hidden_width if k < self.hidden_layers else self.output_width
            shapes.append((out, fin))
            fin = out
        return shapes

    def parameter_count(self) -> int:
        return sum(o * i + o for o, i in self.layer_shapes())


@dataclass
class AdamHyper:   # adam.hpp:13-25
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.99
    eps: float = 1e-15
    l2: float = 1e-6

    def c(self) -> L.nfg_adam_hyper:
        return L.nfg_adam_hyper(self.lr, self.beta1, self.beta2, self.eps, self.l2)


@dataclass
class LrSchedule:   # adam.hpp:124-137
    milestones: List[int] = field(default_factory=list)
    factor: float = 0.33

    def validate(self) -> None:
        if not (self.factor > 0) or self.factor > 1:
            raise ValueError("LrSchedule: factor must be in (0, 1]")
        for a, b in zip(self.milestones, self.milestones[1:]):
            if b <= a:
                raise ValueError("LrSchedule: milestones must be strictly increasing")


def lr_at(schedule: LrSchedule, base_lr: float, step: int) -> float:   # adam.hpp:139-146
    ms = (C.c_int64 * max(len(schedule.milestones), 1))(*schedule.milestones)
    return L.load().nfg_lr_at(ms, len(schedule.milestones), schedule.factor, base_lr, step)


def default_schedule(total_steps: int, factor: float = 0.33) -> LrSchedule:   # adam.hpp:150-161
    s = LrSchedule(factor=factor)
    nxt, stride = int(0.65 * total_steps), int(0.30 * total_steps)
    while nxt < total_steps and stride > 0:
        s.milestones.append(nxt)
        nxt += stride
    return s


@dataclass
class Options:
    """sm_100a build options (no reference equivalent)."""
    table_fp32: bool = False    # gather fp32 master tables instead of the fp16 shadow
    fused_train: bool = True    # one fused kernel per step vs staged encode / MLP / encode-bwd kernels
    deterministic: bool = False  # bit-reproducible backward in the reference's accumulation order
    mlp_engine: int = 0         # 0: measured-faster tensor-core engine per kernel, 1: mma.sync, 2: tcgen05
    dp_exchange: int = 0        # 0/1: chunked all-reduce pipelined with Adam, 2: level-pipelined scatter + exchange

    def c(self) -> L.nfg_options:
        return L.nfg_options(int(self.table_fp32), int(self.fused_train), int(self.deterministic),
                             int(self.mlp_engine), int(self.dp_exchange))


class Context:
    """One CUDA device + stream (+ optional NCCL communicator)."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = C.c_void_p()
        L.check(self.lib.nfg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.nfg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self) -> None:
        L.check(self.lib.nfg_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return int(self.lib.nfg_ctx_stream(self.h) or 0)

    @property
    def launch_count(self) -> int:
        return int(self.lib.nfg_ctx_launch_count(self.h))

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        L.check(L.load().nfg_comm_unique_id(buf))
        return bytes(buf)

    def attach_comm(self, uid: bytes, rank: int, nranks: int) -> None:
        buf = (C.c_uint8 * 128)(*uid)
        L.check(self.lib.nfg_ctx_attach_comm(self.h, buf, rank, nranks))

    def comm_info(self):
        """(rank, nranks) as the attached NCCL communicator reports them."""
        r, n = C.c_int(), C.c_int()
        L.check(self.lib.nfg_ctx_comm_info(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value

    def l2_peak(self, op: int) -> float:
        """Measured L2-level rate of one access kind (diag.cu): 0 random 4 B
        ld.cg, 1 random 4 B cp.async, 2 random red.v2.f32, 4 random 4 B
        ld.nc — sectors/s; 3 streaming L2 reads — bytes/s."""
        r = C.c_double()
        L.check(self.lib.nfg_diag_l2_peak(self.h, op, C.byref(r)))
        return r.value


_DEFAULT_CTX: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dptr(t, what: str = "tensor", dtype: str = "float32") -> Optional[int]:
    """Device pointer of a torch CUDA tensor (or a raw int, taken as is).
    Tensors must be CUDA, contiguous and of the expected dtype: the library
    reads them as flat arrays."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    import torch
    if not t.is_cuda:
        raise L.NfgInvalidArgument(L.NFG_EINVAL, f"{what}: expected a CUDA tensor")
    if t.dtype != getattr(torch, dtype):
        raise L.NfgInvalidArgument(L.NFG_EINVAL, f"{what}: expected dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise L.NfgInvalidArgument(L.NFG_EINVAL, f"{what}: expected a contiguous tensor")
    return int(t.data_ptr())


class _StreamOrder:
    """Orders the library's stream against torch's current stream around a
    device-pointer call: the library waits for torch's pending writes of the
    inputs, and torch's stream waits for the library before it reads the
    outputs or its caching allocator reuses any of the buffers. A no-op when
    no torch tensor is involved (raw pointers: the caller orders)."""

    _ext = {}

    def __init__(self, ctx: "Context", *tensors):
        self.ctx = ctx
        self.on = any(t is not None and not isinstance(t, int) for t in tensors)

    def __enter__(self):
        if self.on:
            import torch
            key = (self.ctx.device, self.ctx.stream)
            ext = _StreamOrder._ext.get(key)
            if ext is None:
                ext = _StreamOrder._ext[key] = torch.cuda.ExternalStream(self.ctx.stream, device=self.ctx.device)
            self.lib_stream = ext
            self.torch_stream = torch.cuda.current_stream(self.ctx.device)
            if self.torch_stream.cuda_stream != ext.cuda_stream:
                ev = torch.cuda.Event()
                ev.record(self.torch_stream)
                ext.wait_event(ev)
        return self

    def __exit__(self, *exc):
        if self.on and self.torch_stream.cuda_stream != self.lib_stream.cuda_stream:
            import torch
            ev = torch.cuda.Event()
            ev.record(self.lib_stream)
            self.torch_stream.wait_event(ev)
        return False


BUF_PARAMS, BUF_GRADS, BUF_ADAM_M, BUF_ADAM_V = range(4)


@dataclass
class EncodeCache:   # grid.hpp:183-195 (exported for checks; the GPU path recomputes)
    rows: np.ndarray
    weights: np.ndarray


class FieldModel:
    """model.hpp:21-63 on the GPU (hash encoder)."""

    def __init__(self, ctx: Optional[Context] = None, options: Optional[Options] = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.hash_cfg = HashEncodingConfig()
        self.mlp_cfg = MlpConfig()
        self.hyper = AdamHyper()
        self.schedule = LrSchedule()
        self.options = options or Options()
        self.h = None
        self._sizes = (0, 0, 0)

    # ---- lifecycle ----------------------------------------------------------
    def _create(self) -> None:
        if self.h:
            self.lib.nfg_field_destroy(self.h)
            self.h = None
        self.mlp_cfg.input_width = self.encoded_width()   # model.cpp:101
        h = C.c_void_p()
        L.check(self.lib.nfg_field_create(self.ctx.h, C.byref(self.hash_cfg.c()), C.byref(self.mlp_cfg.c()),
                                          C.byref(self.hyper.c()), C.byref(self.options.c()), C.byref(h)))
        self.h = h
        sz = (C.c_uint64 * 3)()
        L.check(self.lib.nfg_field_sizes(self.h, sz))
        self._sizes = tuple(int(x) for x in sz)

    def init(self, seed: int) -> None:   # model.cpp:23-37
        self._create()
        L.check(self.lib.nfg_field_init(self.h, seed))
        self._push_schedule()

    def close(self) -> None:
        if self.h:
            self.lib.nfg_field_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _push_schedule(self) -> None:
        self.schedule.validate()
        ms = (C.c_int64 * max(len(self.schedule.milestones), 1))(*self.schedule.milestones)
        L.check(self.lib.nfg_field_set_schedule(self.h, ms, len(self.schedule.milestones), self.schedule.factor))
        L.check(self.lib.nfg_field_set_hyper(self.h, C.byref(self.hyper.c())))

    def encoded_width(self) -> int:
        return self.hash_cfg.output_width()

    def parameter_count(self) -> int:
        return sum(self._sizes)

    @property
    def sizes(self):
        """(table params, MLP weights, MLP biases) — the three param groups."""
        return self._sizes

    # ---- host mirrors of the public members ------------------------------------
    def read(self, which: int, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
        n = self.parameter_count() - offset if count is None else count
        out = np.empty(n, np.float32)
        L.check(self.lib.nfg_field_read(self.h, which, offset, n, _ptr(out)))
        return out

    def write(self, which: int, data, offset: int = 0) -> None:
        d = _f32(data).ravel()
        L.check(self.lib.nfg_field_write(self.h, which, offset, d.size, _ptr(d)))

    @property
    def params(self) -> np.ndarray:
        return self.read(BUF_PARAMS)

    @property
    def grads(self) -> np.ndarray:
        return self.read(BUF_GRADS)

    @property
    def table_params(self) -> np.ndarray:
        return self.read(BUF_PARAMS, 0, self._sizes[0])

    @table_params.setter
    def table_params(self, v) -> None:
        self.write(BUF_PARAMS, v, 0)

    def mlp_weights(self) -> List[np.ndarray]:
        """Weights as (out, in) matrices (the reference's MlpParams::weights)."""
        flat = self.read(BUF_PARAMS, self._sizes[0], self._sizes[1])
        mats, off = [], 0
        for o, i in self.mlp_cfg.layer_shapes():
            mats.append(flat[off: off + o * i].reshape(i, o).T.copy())
            off += o * i
        return mats

    def device_buffer(self, which: int):
        p = L._fp()
        n = C.c_uint64()
        L.check(self.lib.nfg_field_device_buffer(self.h, which, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, int(n.value)

    @property
    def step(self) -> int:
        s = C.c_uint64()
        L.check(self.lib.nfg_field_get_step(self.h, C.byref(s)))
        return int(s.value)

    @step.setter
    def step(self, s: int) -> None:
        L.check(self.lib.nfg_field_set_step(self.h, s))

    def broadcast(self, root: int = 0) -> None:
        """Data parallelism: take root's params, Adam m/v and step (no-op on one rank)."""
        L.check(self.lib.nfg_field_broadcast(self.h, root))

    def adam_state(self):
        """(step, m, v) flat in param-group order (AdamState, adam.hpp:56-73)."""
        return self.step, self.read(BUF_ADAM_M), self.read(BUF_ADAM_V)

    def param_groups(self):
        """The three groups of model.cpp:49-77: (name, offset, size, apply_l2, skip_zero_grad)."""
        t, w, b = self._sizes
        return [("tables", 0, t, False, True), ("mlp_weights", t, w, True, False),
                ("mlp_biases", t + w, b, False, False)]

    # ---- the hot path ----------------------------------------------------------
    def _check_x(self, X) -> np.ndarray:
        X = _f32(X)
        if X.ndim != 2 or X.shape[1] != self.hash_cfg.dims:
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "encode_forward: input dimensionality mismatch")
        # grid.hpp:226-229 — validated on the host like the reference
        if not np.isfinite(X).all():
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "encode_forward: non-finite input")
        if (X < np.float32(-1e-6)).any() or (X > np.float32(1) + np.float32(1e-6)).any():
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "encode_forward: input outside [0,1]^d")
        return X

    def train_step(self, X, target, loss: LossKind, step: int) -> float:   # model.cpp:111-138
        X = self._check_x(X)
        T = _f32(target)
        if T.shape != (X.shape[0], self.mlp_cfg.output_width):
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "l2_loss: shape mismatch")
        self._push_schedule()
        out = C.c_float()
        L.check(self.lib.nfg_field_train_step(self.h, _ptr(X), _ptr(T), X.shape[0], int(loss), step, C.byref(out)))
        return float(out.value)

    def gradients(self, X, target, loss: LossKind) -> float:
        """Forward + loss + backward without Adam; grads accumulate (call adam_step after)."""
        X = self._check_x(X)
        T = _f32(target)
        if T.shape != (X.shape[0], self.mlp_cfg.output_width):
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "l2_loss: shape mismatch")
        out = C.c_float()
        L.check(self.lib.nfg_field_gradients(self.h, _ptr(X), _ptr(T), X.shape[0], int(loss), C.byref(out)))
        return float(out.value)

    def train_step_host_ptr(self, x_ptr: int, t_ptr: int, B: int, loss: LossKind, step: int,
                            B_global: Optional[int] = None) -> float:
        """train_step on caller-owned host buffers (pinned or pageable), no
        validation copy. ``B_global`` (data parallelism, ragged shards): the
        global batch the loss is normalised by; default B x ranks."""
        out = C.c_float()
        if B_global is None:
            L.check(self.lib.nfg_field_train_step(self.h, x_ptr, t_ptr, B, int(loss), step, C.byref(out)))
        else:
            L.check(self.lib.nfg_field_train_step_global(self.h, x_ptr, t_ptr, B, B_global, int(loss), step,
                                                         C.byref(out)))
        return float(out.value)

    def train_step_device(self, X, target, B_local: int, B_global: int, loss: LossKind, step: int,
                          loss_out=None) -> None:
        """Asynchronous step on device pointers (torch CUDA tensors or ints),
        stream-ordered against torch's current stream. ``loss_out`` (optional,
        one float on the device) receives the step's loss; deferred errors are
        reported by check()."""
        with _StreamOrder(self.ctx, X, target, loss_out):
            L.check(self.lib.nfg_field_train_step_device(self.h, _dptr(X, "X"), _dptr(target, "target"), B_local,
                                                         B_global, int(loss), step, _dptr(loss_out, "loss_out")))

    def check(self) -> None:
        L.check(self.lib.nfg_field_check(self.h))

    def last_kernel_variant(self, which: int = 0) -> str:
        """Template instantiation of the last fused train (0) / inference (1)
        kernel launched by this thread (diagnostics; no reference equivalent)."""
        return self.lib.nfg_last_kernel_variant(which).decode()

    def evaluate(self, X) -> np.ndarray:   # model.cpp:102-109
        X = self._check_x(X)
        out = np.empty((X.shape[0], self.mlp_cfg.output_width), np.float32)
        L.check(self.lib.nfg_field_evaluate(self.h, _ptr(X), X.shape[0], _ptr(out)))
        return out

    def evaluate_device(self, X, B: int, out) -> None:
        with _StreamOrder(self.ctx, X, out):
            L.check(self.lib.nfg_field_evaluate_device(self.h, _dptr(X, "X"), B, _dptr(out, "out")))

    # ---- components -------------------------------------------------------------
    def encode_forward(self, X, want_cache: bool = False):   # grid.hpp:219-272
        X = self._check_x(X)
        B = X.shape[0]
        Y = np.empty((B, self.encoded_width()), np.float32)
        rows = wts = None
        if want_cache:
            nc = 1 << self.hash_cfg.dims
            rows = np.empty((self.hash_cfg.levels, B, nc), np.uint32)
            wts = np.empty((self.hash_cfg.levels, B, nc), np.float32)
        L.check(self.lib.nfg_encode_forward(self.h, _ptr(X), B, _ptr(Y), _ptr(rows), _ptr(wts)))
        return (Y, EncodeCache(rows, wts)) if want_cache else Y

    def encode_backward(self, X, dY) -> None:   # grid.hpp:277-295
        X = self._check_x(X)
        dY = _f32(dY)
        if dY.shape != (X.shape[0], self.encoded_width()):
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "encode_backward: gradient shape does not match cache")
        L.check(self.lib.nfg_encode_backward(self.h, _ptr(X), X.shape[0], _ptr(dY)))

    def mlp_forward(self, Y) -> np.ndarray:   # mlp.hpp:104-124
        Y = _f32(Y)
        if Y.ndim != 2 or Y.shape[1] != self.mlp_cfg.input_width:
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "mlp_forward: input width mismatch")
        out = np.empty((Y.shape[0], self.mlp_cfg.output_width), np.float32)
        L.check(self.lib.nfg_mlp_forward(self.h, _ptr(Y), Y.shape[0], _ptr(out)))
        return out

    def mlp_backward(self, Y, dOut) -> np.ndarray:   # mlp.hpp:129-158 (grads accumulate)
        Y = _f32(Y)
        dOut = _f32(dOut)
        if dOut.shape != (Y.shape[0], self.mlp_cfg.output_width):
            raise L.NfgInvalidArgument(L.NFG_EINVAL, "mlp_backward: shape mismatch with cache")
        dY = np.empty((Y.shape[0], self.mlp_cfg.input_width), np.float32)
        L.check(self.lib.nfg_mlp_backward(self.h, _ptr(Y), Y.shape[0], _ptr(dOut), _ptr(dY)))
        return dY

    def adam_step(self, lr_now: float) -> None:   # adam.hpp:78-122 over param_groups()
        L.check(self.lib.nfg_adam_step(self.h, C.c_float(lr_now)))


def loss_with_grad(kind: LossKind, pred, target, ctx: Optional[Context] = None):   # model.cpp:140-149
    p = _f32(pred)
    t = _f32(target)
    if p.shape != t.shape:
        raise L.NfgInvalidArgument(L.NFG_EINVAL, "l2_loss: shape mismatch")
    ctx = ctx or default_context()
    d = np.empty_like(p)
    out = C.c_float()
    L.check(ctx.lib.nfg_loss(ctx.h, int(kind), _ptr(p), _ptr(t), p.size, p.size, _ptr(d), C.byref(out)))
    return float(out.value), d


# ---- checkpoint + train report (io.cpp:189-351) --------------------------------
def save_checkpoint(model: "FieldModel", path: str) -> None:   # io.cpp:222-285
    """NFC1/HGE1/MLP1/ADM1 bytes, loadable by the reference's load_checkpoint."""
    L.check(model.lib.nfg_field_save(model.h, os.fsencode(path)))


def load_checkpoint(model: "FieldModel", path: str) -> None:   # io.cpp:287-351
    """Replaces the model's configs, parameters and Adam state with the file's;
    ``model.hyper`` / ``schedule`` / ``options`` are kept (re-supplied by the
    caller on resume, test_tasks.cpp:313-315)."""
    h = C.c_void_p()
    L.check(model.lib.nfg_field_load(model.ctx.h, os.fsencode(path), C.byref(model.hyper.c()),
                                     C.byref(model.options.c()), C.byref(h)))
    model.close()
    model.h = h
    g, m = L.nfg_grid_config(), L.nfg_mlp_config()
    L.check(model.lib.nfg_field_get_config(h, C.byref(g), C.byref(m)))
    model.hash_cfg = HashEncodingConfig(g.levels, g.table_size, g.features, g.n_min, g.n_max, g.dims,
                                        Interpolation(g.interpolation))
    model.mlp_cfg = MlpConfig(m.input_width, m.hidden_layers, m.hidden_width, m.output_width,
                              OutputActivation(m.output_activation))
    sz = (C.c_uint64 * 3)()
    L.check(model.lib.nfg_field_sizes(h, sz))
    model._sizes = tuple(int(x) for x in sz)
    model._push_schedule()


@dataclass
class TrainReportRow:   # io.hpp:25-31
    step: int = 0
    time_s: float = 0.0
    loss: float = 0.0
    metric: float = 0.0
    lr: float = 0.0


@dataclass
class TrainReport:   # io.hpp:33-35
    rows: List[TrainReportRow] = field(default_factory=list)


def _g10(v) -> str:
    """C++ ostream with precision(10) (default float format) == printf %.10g."""
    return "%.10g" % v


def write_report_csv(report: TrainReport, path: str) -> None:   # io.cpp:189-199
    try:
        with open(path, "w") as out:
            out.write("step,time_s,loss,metric,lr\n")
            for r in report.rows:
                out.write(f"{int(r.step)},{_g10(r.time_s)},{_g10(r.loss)},{_g10(r.metric)},{_g10(r.lr)}\n")
    except OSError:
        raise L.NfgIOError(L.NFG_EIO, "cannot write report: " + path) from None


def read_report_csv(path: str) -> TrainReport:   # io.cpp:201-220
    try:
        with open(path) as f:
            lines = f.read().splitlines()
    except OSError:
        raise L.NfgIOError(L.NFG_EIO, "cannot read report: " + path) from None
    rep = TrainReport()
    for line in lines[1:]:
        if not line:
            continue
        a = line.split(",")
        rep.rows.append(TrainReportRow(int(a[0]), float(a[1]), float(a[2]), float(a[3]), float(a[4])))
    return rep


# ---- training-loop data path on the device (tasks.cpp) -------
class DeviceRng:
    """Pcg32(seed, seq) (pcg32.hpp) as a device stream: ``below`` / ``floats``
    fill device buffers (torch CUDA tensors or pointers) with exactly the draws
    of n sequential host calls (rejection sampling included)."""

    def __init__(self, seed: int, seq: int = 1, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        h = C.c_void_p()
        L.check(self.lib.nfg_rng_create(self.ctx.h, seed, seq, C.byref(h)))
        self.h = h

    def below(self, bound: int, n: int, out) -> None:   # next_below x n (pcg32.hpp:30-38)
        with _StreamOrder(self.ctx, out):
            L.check(self.lib.nfg_rng_below_device(self.h, bound, n, _dptr(out, "out", "int32")))

    def floats(self, n: int, out) -> None:   # next_float x n (pcg32.hpp:41-44)
        with _StreamOrder(self.ctx, out):
            L.check(self.lib.nfg_rng_floats_device(self.h, n, _dptr(out, "out")))

    def state(self):
        s, i = C.c_uint64(), C.c_uint64()
        L.check(self.lib.nfg_rng_get_state(self.h, C.byref(s), C.byref(i)))
        return int(s.value), int(i.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.nfg_rng_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ImageTask:   # tasks.hpp:16-31 (hash encoder)
    image: np.ndarray = None          # (w*h, 3) float32, pixel i = y*w + x (Image::rgb, io.hpp:12-19)
    width: int = 0
    height: int = 0
    cfg: HashEncodingConfig = field(default_factory=lambda: HashEncodingConfig(n_max=0))   # n_max <= 0: width/2
    interpolation: Interpolation = Interpolation.Linear
    hidden_layers: int = 2
    hidden_width: int = 64
    batch_size: int = 1 << 14
    total_steps: int = 10000
    log_interval: int = 1000
    lr: float = 1e-2
    lr_decay: float = 0.33


@dataclass
class SdfTask:   # tasks.hpp:33-50 (hash encoder; analytic CSG target instead of a mesh)
    cfg: HashEncodingConfig = field(default_factory=HashEncodingConfig)
    hidden_layers: int = 2
    hidden_width: int = 64
    batch_size: int = 1 << 13
    total_steps: int = 10000
    log_interval: int = 1000
    lr: float = 1e-4
    lr_decay: float = 0.33
    loss: LossKind = LossKind.Mape
    iou_eval_points: int = 1 << 16


@dataclass
class FitResult:   # tasks.hpp:58-61
    model: "FieldModel"
    report: TrainReport


def fit_image(task: ImageTask, seed: int, options: Optional[Options] = None,
              ctx: Optional[Context] = None) -> FitResult:   # tasks.cpp:49-131, all steps on the device
    ctx = ctx or default_context()
    rgb = _f32(task.image)
    if rgb.shape != (task.width * task.height, 3):
        raise L.NfgInvalidArgument(L.NFG_EINVAL, "fit_image: image shape does not match width x height")
    cfg = HashEncodingConfig(task.cfg.levels, task.cfg.table_size, task.cfg.features, task.cfg.n_min,
                             task.cfg.n_max, 2, task.interpolation)
    t = L.nfg_image_task(task.width, task.height, cfg.c(), task.hidden_layers, task.hidden_width, task.batch_size,
                         task.total_steps, task.log_interval, task.lr, task.lr_decay)
    cap = task.total_steps // max(task.log_interval, 1) + 2
    rows = (L.nfg_report_row * cap)()
    n = C.c_int64()
    h = C.c_void_p()
    opts = options or Options()
    L.check(ctx.lib.nfg_fit_image(ctx.h, C.byref(t), _ptr(rgb), seed, C.byref(opts.c()), C.byref(h), rows, cap,
                                  C.byref(n)))
    model = _adopt_field(ctx, h, opts, task.lr, task.total_steps, task.lr_decay)
    rep = TrainReport([TrainReportRow(int(r.step), r.time_s, r.loss, r.metric, r.lr)
                       for r in rows[:min(n.value, cap)]])
    return FitResult(model, rep)


# ---- inference consumers (tasks.cpp:195-356) -----------------
@dataclass
class Camera:   # tasks.hpp:72-77
    position: tuple = (0.5, 0.5, -1.2)
    target: tuple = (0.5, 0.5, 0.5)
    up: tuple = (0.0, 1.0, 0.0)
    fov_deg: float = 40.0

    def c(self) -> L.nfg_camera:
        return L.nfg_camera((C.c_double * 3)(*self.position), (C.c_double * 3)(*self.target),
                            (C.c_double * 3)(*self.up), self.fov_deg)


def _field_args(field, dims: int):
    """(nfg_field handle, FieldFn callback) for a FieldModel or a Python callable
    mapping an (n, dims) float32 array to n values."""
    if isinstance(field, FieldModel):
        return field.h, L.FIELD_FN(), field.ctx

    def cb(xp, n, outp, _user):
        X = np.ctypeslib.as_array(xp, shape=(int(n), dims))
        out = np.ctypeslib.as_array(outp, shape=(int(n),))
        out[:] = np.asarray(field(X), np.float32).reshape(-1)[: int(n)]

    return None, L.FIELD_FN(cb), None


def render_image(model: "FieldModel", width: int, height: int) -> np.ndarray:   # tasks.cpp:195-209
    """(width*height, output_width) float32, pixel i = y*width + x."""
    out = np.empty((width * height, model.mlp_cfg.output_width), np.float32)
    L.check(model.lib.nfg_render_image(model.h, width, height, _ptr(out)))
    return out


def render_sdf_shaded(field, camera: Camera, width: int, height: int,
                      ctx: Optional[Context] = None) -> np.ndarray:   # tasks.cpp:233-329
    """Sphere-traced, Lambert-shaded image of the zero level set: (width*height, 3)."""
    h, fn, fctx = _field_args(field, 3)
    ctx = fctx or ctx or default_context()
    out = np.empty((width * height, 3), np.float32)
    L.check(ctx.lib.nfg_render_sdf_shaded(ctx.h, h, fn, None, C.byref(camera.c()), width, height, _ptr(out)))
    return out


def iou(field, oracle_sign, n_points: int, rng: DeviceRng, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)) -> float:
    """tasks.cpp:331-356: ``oracle_sign(p)`` gets a (3,) float64 point; points come
    from ``rng`` exactly as Pcg32::uniform<double>."""
    h, fn, _ = _field_args(field, 3)

    def sign(pp, _user):
        return int(oracle_sign(np.ctypeslib.as_array(pp, shape=(3,)).copy()))

    scb = L.SIGN_FN(sign)
    out = C.c_double()
    L.check(rng.lib.nfg_iou(rng.ctx.h, h, fn, None, scb, None, n_points, rng.h, (C.c_double * 3)(*lo),
                            (C.c_double * 3)(*hi), C.byref(out)))
    return float(out.value)


# ---- NeRF (§5.4 + Appendix E) -------------------------
OCC_RES = 128


def orbit_cameras(n: int, radius: float = 1.3, height: float = 0.25, fov_deg: float = 40.0, width: int = 64,
                  phase: float = 0.0):
    """n views on a circle around (0.5, 0.5, 0.5) looking at the centre: (cams (n, 12), focal)."""
    cams = np.zeros((n, 12), np.float32)
    for i in range(n):
        a = phase + 2 * np.pi * i / n
        pos = np.array([0.5 + radius * np.cos(a), 0.5 + height * np.sin(3 * a + 0.3), 0.5 + radius * np.sin(a)])
        fwd = np.array([0.5, 0.5, 0.5]) - pos
        fwd /= np.linalg.norm(fwd)
        right = np.cross(fwd, [0.0, 1.0, 0.0])
        right /= np.linalg.norm(right)
        up = np.cross(right, fwd)
        cams[i] = np.concatenate([pos, fwd, right, up]).astype(np.float32)
    focal = 0.5 * width / np.tan(0.5 * np.radians(fov_deg))
    return cams, float(focal)


class NeRF:
    """Hash-grid NeRF (density 1x64 -> 16, color 2x64 -> RGB) trained with
    occupancy-grid ray marching and compacted samples, all on the device."""

    def __init__(self, grid: Optional[HashEncodingConfig] = None, lr: float = 1e-2, target_samples: int = 1 << 18,
                 max_samples_per_ray: int = 1024, background=(1.0, 1.0, 1.0), seed: int = 1337,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        g = grid or HashEncodingConfig(levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, dims=3)
        cfg = L.nfg_nerf_config(g.c(), lr, target_samples, max_samples_per_ray, (C.c_float * 3)(*background))
        h = C.c_void_p()
        L.check(self.lib.nfg_nerf_create(self.ctx.h, C.byref(cfg), seed, C.byref(h)))
        self.h = h
        self.background = tuple(background)

    def set_dataset(self, cams, rgb, width: int, height: int, focal: float) -> None:
        cams = _f32(cams)
        rgb = _f32(rgb)
        self._keep = (cams, rgb)
        L.check(self.lib.nfg_nerf_set_dataset(self.h, cams.shape[0], width, height, focal, _ptr(cams), _ptr(rgb)))

    def train_step(self, step: int):
        """-> (loss, rays used, samples marched); ``last_backward_samples`` holds the
        samples that reached the backward networks (before the transmittance stop)."""
        loss, nr, ns, nb = C.c_float(), C.c_int64(), C.c_int64(), C.c_int64()
        L.check(self.lib.nfg_nerf_train_step2(self.h, step, C.byref(loss), C.byref(nr), C.byref(ns), C.byref(nb)))
        self.last_backward_samples = int(nb.value)
        return float(loss.value), int(nr.value), int(ns.value)

    def render(self, cam, width: int, height: int, focal: float) -> np.ndarray:
        cam = _f32(cam).reshape(12)
        out = np.empty((height * width, 3), np.float32)
        L.check(self.lib.nfg_nerf_render(self.h, _ptr(cam), width, height, focal, _ptr(out)))
        return out

    def sync(self) -> None:
        """Apply the Adam step the last train_step deferred and wait for the GPU."""
        L.check(self.lib.nfg_nerf_sync(self.h))

    def occupancy(self):
        bits = np.empty(OCC_RES ** 3 // 8, np.uint8)
        dens = np.empty(OCC_RES ** 3, np.float32)
        L.check(self.lib.nfg_nerf_occupancy(self.h, _ptr(bits), _ptr(dens)))
        return bits, dens

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.nfg_nerf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nerf_march(rays, bits, max_steps: int = 1024, ctx: Optional[Context] = None):
    """Occupancy-grid marching + compaction: (counts (n,), samples (total, 3))."""
    ctx = ctx or default_context()
    rays = _f32(rays)
    bits = np.ascontiguousarray(bits, np.uint8)
    n = rays.shape[0]
    counts = np.zeros(n, np.uint32)
    cap = n * max_steps
    samples = np.empty((max(cap, 1), 3), np.float32)
    tot = C.c_int64()
    L.check(ctx.lib.nfg_nerf_march(ctx.h, _ptr(rays), n, _ptr(bits), max_steps, _ptr(counts), _ptr(samples), cap,
                                   C.byref(tot)))
    return counts, samples[: tot.value].copy()


def nerf_composite(counts, raw, rgb, target, bg=(1.0, 1.0, 1.0), dt: float = 3 ** 0.5 / 1024,
                   ctx: Optional[Context] = None):
    """Compositing forward + backward: (color (R,3), d_rgb (S,3), d_raw (S,), loss_sum)."""
    ctx = ctx or default_context()
    counts = np.ascontiguousarray(counts, np.uint32)
    raw, rgb, target = _f32(raw), _f32(rgb), _f32(target)
    R, S = counts.shape[0], raw.shape[0]
    color = np.empty((R, 3), np.float32)
    d_rgb = np.empty((S, 3), np.float32)
    d_raw = np.empty(S, np.float32)
    bgv = np.asarray(bg, np.float32)
    loss = C.c_double()
    L.check(ctx.lib.nfg_nerf_composite(ctx.h, R, _ptr(counts), _ptr(raw), _ptr(rgb), _ptr(target), _ptr(bgv), dt,
                                       _ptr(color), _ptr(d_rgb), _ptr(d_raw), C.byref(loss)))
    return color, d_rgb, d_raw, float(loss.value)


def nerf_sh4(dirs, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    dirs = _f32(dirs)
    out = np.empty((dirs.shape[0], 16), np.float32)
    L.check(ctx.lib.nfg_nerf_sh4(ctx.h, _ptr(dirs), dirs.shape[0], _ptr(out)))
    return out


def nerf_scene_render(cams, width: int, height: int, focal: float, bg=(1.0, 1.0, 1.0),
                      ctx: Optional[Context] = None) -> np.ndarray:
    """The synthetic procedural scene (BASELINE config 4) by fine marching: (n, h*w, 3)."""
    ctx = ctx or default_context()
    cams = _f32(cams)
    out = np.empty((cams.shape[0], height * width, 3), np.float32)
    bgv = np.asarray(bg, np.float32)
    L.check(ctx.lib.nfg_nerf_scene_render(ctx.h, _ptr(cams), cams.shape[0], width, height, focal, _ptr(bgv),
                                          _ptr(out)))
    return out


def _adopt_field(ctx: Context, h, opts: "Options", lr: float, total_steps: int, lr_decay: float) -> "FieldModel":
    model = FieldModel(ctx, opts)
    model.h = h
    g, m = L.nfg_grid_config(), L.nfg_mlp_config()
    L.check(ctx.lib.nfg_field_get_config(h, C.byref(g), C.byref(m)))
    model.hash_cfg = HashEncodingConfig(g.levels, g.table_size, g.features, g.n_min, g.n_max, g.dims,
                                        Interpolation(g.interpolation))
    model.mlp_cfg = MlpConfig(m.input_width, m.hidden_layers, m.hidden_width, m.output_width,
                              OutputActivation(m.output_activation))
    model.hyper = AdamHyper(lr=lr)
    model.schedule = default_schedule(total_steps, lr_decay)
    sz = (C.c_uint64 * 3)()
    L.check(ctx.lib.nfg_field_sizes(h, sz))
    model._sizes = tuple(int(x) for x in sz)
    return model


def fit_sdf_analytic(task: SdfTask, seed: int, options: Optional[Options] = None,
                     ctx: Optional[Context] = None) -> FitResult:   # tasks.cpp:133-193 on the config-2 CSG target
    ctx = ctx or default_context()
    g = task.cfg
    cfg = HashEncodingConfig(g.levels, g.table_size, g.features, g.n_min, g.n_max, 3, g.interpolation)
    t = L.nfg_sdf_task(cfg.c(), task.hidden_layers, task.hidden_width, task.batch_size, int(task.loss),
                       task.total_steps, task.log_interval, task.iou_eval_points, task.lr, task.lr_decay)
    cap = task.total_steps // max(task.log_interval, 1) + 2
    rows = (L.nfg_report_row * cap)()
    n = C.c_int64()
    h = C.c_void_p()
    opts = options or Options()
    L.check(ctx.lib.nfg_fit_sdf_analytic(ctx.h, C.byref(t), seed, C.byref(opts.c()), C.byref(h), rows, cap,
                                         C.byref(n)))
    model = _adopt_field(ctx, h, opts, task.lr, task.total_steps, task.lr_decay)
    rep = TrainReport([TrainReportRow(int(r.step), r.time_s, r.loss, r.metric, r.lr) for r in rows[:min(n.value, cap)]])
    return FitResult(model, rep)


class PinnedBuffer:
    """Page-locked host memory (cudaMallocHost) viewed as a numpy array."""

    def __init__(self, shape, dtype=np.float32):
        self.lib = L.load()
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        L.check(self.lib.nfg_host_alloc(max(nbytes, 1), C.byref(p)))
        self.ptr = p.value
        buf = (C.c_uint8 * nbytes).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def free(self) -> None:
        if getattr(self, "ptr", None):
            self.lib.nfg_host_free(C.c_void_p(self.ptr))
            self.ptr = None
