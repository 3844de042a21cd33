"""Experiment: k_train time on random vs spatially ordered batches (config 2).

Measures the potential of sorting each batch by coarse cell before the fused
kernel (L1 locality of coarse-level gathers, same-row reductions within a warp).
Usage (GPU): python tools/exp_sort.py
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CFG2, sdf_torch  # noqa: E402
from paper_2201_05989_b200 import nf  # noqa: E402

B = 1 << 18


def morton_key(X, bits):
    c = (X.clamp(0, 1 - 1e-7) * (1 << bits)).long()
    key = torch.zeros(X.shape[0], dtype=torch.long, device=X.device)
    for b in range(bits):
        for d in range(3):
            key |= ((c[:, d] >> b) & 1) << (3 * b + d)
    return key


def run(model, Xs, Ts, steps=30):
    ctx = model.ctx
    lib = ctx.lib
    for i in range(5):
        model.train_step_device(Xs[i % len(Xs)], Ts[i % len(Xs)], B, B, nf.LossKind.Mape, i + 1)
    ctx.synchronize()
    lib.nfg_ctx_set_profiling(ctx.h, 1)
    ms = (C.c_double * 4)()
    n = C.c_int64()
    lib.nfg_ctx_read_profile(ctx.h, ms, C.byref(n))
    for i in range(steps):
        model.train_step_device(Xs[i % len(Xs)], Ts[i % len(Xs)], B, B, nf.LossKind.Mape, 10 + i)
    ctx.synchronize()
    lib.nfg_ctx_read_profile(ctx.h, ms, C.byref(n))
    lib.nfg_ctx_set_profiling(ctx.h, 0)
    return ms[0] / steps, ms[1] / steps


def main():
    torch.cuda.set_device(0)
    model = nf.FieldModel()
    model.hash_cfg = nf.HashEncodingConfig(**CFG2)
    model.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
    model.hyper = nf.AdamHyper(lr=1e-4)
    model.init(1337)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    Xs = [torch.rand(B, 3, device="cuda", generator=g) for _ in range(8)]
    Ts = [sdf_torch(x) for x in Xs]
    print("random      k_train %.1f us  adam %.1f us" % tuple(1e3 * v for v in run(model, Xs, Ts)))
    for bits in (3, 4, 5, 6, 8, 10):
        Xo, To = [], []
        for x, t in zip(Xs, Ts):
            p = torch.argsort(morton_key(x, bits))
            Xo.append(x[p].contiguous())
            To.append(t[p].contiguous())
        print("morton%-2d    k_train %.1f us  adam %.1f us" % ((bits,) + tuple(1e3 * v for v in run(model, Xo, To))))


if __name__ == "__main__":
    main()
