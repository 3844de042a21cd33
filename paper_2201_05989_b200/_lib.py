"""ctypes binding of libnfg.so (the sm_100a C ABI declared in include/nfg.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2201_05989_b200``). There is no CPU fallback: if the shared library is
missing or cannot be loaded this module raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NFG_LIB", os.path.join(_HERE, "libnfg.so"))   # NFG_LIB: A/B builds

NFG_OK, NFG_EINVAL, NFG_ENONFINITE, NFG_EUNSUPPORTED, NFG_ECUDA, NFG_ENCCL, NFG_ELOGIC, NFG_EIO = range(8)


class nfg_grid_config(C.Structure):
    _fields_ = [("levels", C.c_int32), ("table_size", C.c_uint32), ("features", C.c_int32),
                ("n_min", C.c_int32), ("n_max", C.c_int32), ("dims", C.c_int32), ("interpolation", C.c_int32)]


class nfg_level_spec(C.Structure):
    _fields_ = [("level", C.c_int32), ("resolution", C.c_uint32), ("table_len", C.c_uint32),
                ("dense", C.c_int32), ("row_offset", C.c_uint64)]


class nfg_mlp_config(C.Structure):
    _fields_ = [("input_width", C.c_int32), ("hidden_layers", C.c_int32), ("hidden_width", C.c_int32),
                ("output_width", C.c_int32), ("output_activation", C.c_int32)]


class nfg_adam_hyper(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("l2", C.c_double)]


class nfg_options(C.Structure):
    _fields_ = [("table_fp32", C.c_int32), ("fused_train", C.c_int32), ("deterministic", C.c_int32),
                ("mlp_engine", C.c_int32), ("dp_exchange", C.c_int32)]


class nfg_image_task(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("cfg", nfg_grid_config),
                ("hidden_layers", C.c_int32), ("hidden_width", C.c_int32), ("batch_size", C.c_int32),
                ("total_steps", C.c_int64), ("log_interval", C.c_int64), ("lr", C.c_double), ("lr_decay", C.c_double)]


class nfg_sdf_task(C.Structure):
    _fields_ = [("cfg", nfg_grid_config), ("hidden_layers", C.c_int32), ("hidden_width", C.c_int32),
                ("batch_size", C.c_int32), ("loss", C.c_int32), ("total_steps", C.c_int64),
                ("log_interval", C.c_int64), ("iou_eval_points", C.c_int64), ("lr", C.c_double),
                ("lr_decay", C.c_double)]


class nfg_report_row(C.Structure):
    _fields_ = [("step", C.c_int64), ("time_s", C.c_double), ("loss", C.c_double), ("metric", C.c_double),
                ("lr", C.c_double)]


class nfg_step_record(C.Structure):
    _fields_ = [("loss_sum", C.c_double), ("flags", C.c_uint32 * 4), ("dy_max", C.c_float), ("pad", C.c_float)]


class nfg_camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("target", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_deg", C.c_double)]


class nfg_nerf_config(C.Structure):
    _fields_ = [("grid", nfg_grid_config), ("lr", C.c_double), ("target_samples", C.c_int32),
                ("max_samples_per_ray", C.c_int32), ("background", C.c_float * 3)]


FIELD_FN = C.CFUNCTYPE(None, C.POINTER(C.c_float), C.c_int64, C.POINTER(C.c_float), C.c_void_p)
SIGN_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_void_p)

_vp = C.c_void_p
_fp = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)

# name -> (restype, argtypes); the authoritative list of exported symbols (include/nfg.h)
SIGNATURES = {
    "nfg_last_error": (C.c_char_p, []),
    "nfg_abi_version": (C.c_int, []),
    "nfg_last_kernel_variant": (C.c_char_p, [C.c_int32]),
    "nfg_diag_l2_peak": (C.c_int, [_vp, C.c_int32, C.POINTER(C.c_double)]),
    "nfg_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "nfg_ctx_destroy": (C.c_int, [_vp]),
    "nfg_ctx_synchronize": (C.c_int, [_vp]),
    "nfg_ctx_stream": (_vp, [_vp]),
    "nfg_ctx_launch_count": (C.c_uint64, [_vp]),
    "nfg_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "nfg_ctx_read_profile": (C.c_int, [_vp, C.POINTER(C.c_double), _i64p]),
    "nfg_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "nfg_ctx_attach_comm": (C.c_int, [_vp, C.POINTER(C.c_uint8), C.c_int, C.c_int]),
    "nfg_ctx_comm_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "nfg_field_broadcast": (C.c_int, [_vp, C.c_int]),
    "nfg_level_resolutions": (C.c_int32, [C.POINTER(nfg_grid_config), C.POINTER(nfg_level_spec), C.c_int32]),
    "nfg_growth_factor": (C.c_double, [C.POINTER(nfg_grid_config)]),
    "nfg_spatial_hash": (C.c_uint32, [_u32p, C.c_int32, C.c_uint32]),
    "nfg_field_create": (C.c_int, [_vp, C.POINTER(nfg_grid_config), C.POINTER(nfg_mlp_config),
                                   C.POINTER(nfg_adam_hyper), C.POINTER(nfg_options), C.POINTER(_vp)]),
    "nfg_field_destroy": (C.c_int, [_vp]),
    "nfg_field_init": (C.c_int, [_vp, C.c_uint64]),
    "nfg_field_set_hyper": (C.c_int, [_vp, C.POINTER(nfg_adam_hyper)]),
    "nfg_field_set_schedule": (C.c_int, [_vp, _i64p, C.c_int32, C.c_double]),
    "nfg_field_sizes": (C.c_int, [_vp, _u64p]),
    "nfg_field_levels": (C.c_int, [_vp, C.POINTER(nfg_level_spec), C.c_int32]),
    "nfg_field_read": (C.c_int, [_vp, C.c_int32, C.c_uint64, C.c_uint64, _vp]),
    "nfg_field_write": (C.c_int, [_vp, C.c_int32, C.c_uint64, C.c_uint64, _vp]),
    "nfg_field_device_buffer": (C.c_int, [_vp, C.c_int32, C.POINTER(_fp), _u64p]),
    "nfg_field_get_config": (C.c_int, [_vp, C.POINTER(nfg_grid_config), C.POINTER(nfg_mlp_config)]),
    "nfg_field_get_step": (C.c_int, [_vp, _u64p]),
    "nfg_field_set_step": (C.c_int, [_vp, C.c_uint64]),
    "nfg_field_train_step": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int64, _fp]),
    "nfg_field_train_step_global": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int64, C.c_int32, C.c_int64, _fp]),
    "nfg_field_train_step_device": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int64, C.c_int32, C.c_int64, _vp]),
    "nfg_field_gradients": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, _fp]),
    "nfg_field_check": (C.c_int, [_vp]),
    "nfg_field_evaluate": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_field_evaluate_device": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_encode_forward": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp, _vp]),
    "nfg_encode_backward": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_mlp_forward": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_mlp_backward": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "nfg_loss": (C.c_int, [_vp, C.c_int32, _vp, _vp, C.c_int64, C.c_int64, _vp, _fp]),
    "nfg_adam_step": (C.c_int, [_vp, C.c_float]),
    "nfg_lr_at": (C.c_double, [_i64p, C.c_int32, C.c_double, C.c_double, C.c_int64]),
    "nfg_field_save": (C.c_int, [_vp, C.c_char_p]),
    "nfg_field_load": (C.c_int, [_vp, C.c_char_p, C.POINTER(nfg_adam_hyper), C.POINTER(nfg_options), C.POINTER(_vp)]),
    "nfg_field_step_record": (C.c_int, [_vp, _vp]),
    "nfg_step_record_check": (C.c_int, [_vp, C.POINTER(nfg_step_record), C.c_int64, _fp]),
    "nfg_rng_create": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.POINTER(_vp)]),
    "nfg_rng_destroy": (C.c_int, [_vp]),
    "nfg_rng_below_device": (C.c_int, [_vp, C.c_uint32, C.c_int64, _vp]),
    "nfg_rng_floats_device": (C.c_int, [_vp, C.c_int64, _vp]),
    "nfg_rng_get_state": (C.c_int, [_vp, _u64p, _u64p]),
    "nfg_image_batch_device": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int32, C.c_int32, _vp, _vp]),
    "nfg_fit_image": (C.c_int, [_vp, C.POINTER(nfg_image_task), _vp, C.c_uint64, C.POINTER(nfg_options),
                                C.POINTER(_vp), C.POINTER(nfg_report_row), C.c_int64, _i64p]),
    "nfg_rng_u32_device": (C.c_int, [_vp, C.c_int64, _vp]),
    "nfg_field_context": (C.c_int, [_vp, C.POINTER(_vp)]),
    "nfg_render_image": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp]),
    "nfg_render_sdf_shaded": (C.c_int, [_vp, _vp, FIELD_FN, _vp, C.POINTER(nfg_camera), C.c_int32, C.c_int32, _vp]),
    "nfg_iou": (C.c_int, [_vp, _vp, FIELD_FN, _vp, SIGN_FN, _vp, C.c_int64, _vp, C.POINTER(C.c_double),
                          C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "nfg_field_backward_device": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_mlp_forward_device": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_mlp_backward_device": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "nfg_adam_step_device": (C.c_int, [_vp, C.c_float]),
    "nfg_nerf_create": (C.c_int, [_vp, C.POINTER(nfg_nerf_config), C.c_uint64, C.POINTER(_vp)]),
    "nfg_nerf_destroy": (C.c_int, [_vp]),
    "nfg_nerf_fields": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
    "nfg_nerf_set_dataset": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_float, _vp, _vp]),
    "nfg_nerf_train_step": (C.c_int, [_vp, C.c_int64, _fp, _i64p, _i64p]),
    "nfg_nerf_train_step2": (C.c_int, [_vp, C.c_int64, _fp, _i64p, _i64p, _i64p]),
    "nfg_nerf_update_occupancy": (C.c_int, [_vp, C.c_int64]),
    "nfg_nerf_sync": (C.c_int, [_vp]),
    "nfg_nerf_render": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_float, _vp]),
    "nfg_nerf_occupancy": (C.c_int, [_vp, _vp, _vp]),
    "nfg_nerf_set_occupancy": (C.c_int, [_vp, _vp]),
    "nfg_nerf_march": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int32, _vp, _vp, C.c_int64, _i64p]),
    "nfg_nerf_composite": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, C.c_float, _vp, _vp, _vp,
                                     C.POINTER(C.c_double)]),
    "nfg_nerf_sh4": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_nerf_scene_render": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_float, _vp, _vp]),
    "nfg_fit_sdf_analytic": (C.c_int, [_vp, C.POINTER(nfg_sdf_task), C.c_uint64, C.POINTER(nfg_options),
                                       C.POINTER(_vp), C.POINTER(nfg_report_row), C.c_int64, _i64p]),
    "nfg_csg_sdf_device": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "nfg_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "nfg_host_free": (C.c_int, [_vp]),
}

_lib = None


class NfgError(RuntimeError):
    """Base error; subclasses mirror the reference's exception types."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class NfgInvalidArgument(NfgError, ValueError):
    """std::invalid_argument"""


class NfgNonFinite(NfgError):
    """std::runtime_error from adam_step (non-finite gradient)"""


class NfgUnsupported(NfgError, NotImplementedError):
    """valid for the reference, not built for sm_100a"""


class NfgIOError(NfgError):
    """std::runtime_error from checkpoint / report IO (io.cpp)"""


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libnfg.so (no fallback: a missing library is an error)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libnfg.so not built at {path}; run __graft_entry__.build() or make -C {_HERE}")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == NFG_OK:
        return
    msg = load().nfg_last_error().decode()
    if status == NFG_EINVAL:
        raise NfgInvalidArgument(status, msg)
    if status == NFG_ENONFINITE:
        raise NfgNonFinite(status, msg)
    if status == NFG_EUNSUPPORTED:
        raise NfgUnsupported(status, msg)
    if status == NFG_EIO:
        raise NfgIOError(status, msg)
    raise NfgError(status, msg)
