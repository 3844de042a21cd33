"""B200-native (sm_100a) multiresolution hash encoding + fully fused MLP + Adam.

A drop-in for the reference's hot path (/root/reference/proj/include/nf/*.hpp):
``nf`` mirrors its API; ``_lib`` binds the C ABI (include/nfg.h) implemented by
the in-tree ``libnfg.so``.
"""
from . import _lib  # noqa: F401
from .nf import (AdamHyper, Context, FieldModel, HashEncodingConfig, Interpolation, LossKind,  # noqa: F401
                 LrSchedule, MlpConfig, Options, OutputActivation, default_schedule, level_resolutions,
                 loss_with_grad, lr_at, spatial_hash)

__all__ = ["AdamHyper", "Context", "FieldModel", "HashEncodingConfig", "Interpolation", "LossKind", "LrSchedule",
           "MlpConfig", "Options", "OutputActivation", "default_schedule", "level_resolutions", "loss_with_grad",
           "lr_at", "spatial_hash"]
