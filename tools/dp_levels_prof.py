"""Config-2 data-parallel step on one GPU through a 1-rank NCCL communicator,
for the launch list of the level-pipelined exchange (run under ncu
--metrics gpu__time_duration.sum) and the step time of each exchange mode.
Usage: python tools/dp_levels_prof.py [steps]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_05989_b200 import nf  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    B = 1 << 18
    X = torch.rand(B, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    c = X - 0.5
    T = (torch.sqrt((c * c).sum(1)) - 0.3).unsqueeze(1).contiguous()
    out = {}
    only = os.environ.get("DP_ONLY")
    for exchange in ((int(only),) if only else (0, 1, 2)):   # none (no communicator), all-reduce, levels
        ctx = nf.Context(0)
        if exchange:
            ctx.attach_comm(nf.Context.unique_id(), 0, 1)
        m = nf.FieldModel(ctx, options=nf.Options(dp_exchange=max(exchange, 1)))
        m.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, dims=3)
        m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
        m.hyper = nf.AdamHyper(lr=1e-4)
        m.init(1337)
        for s in range(1, 4):
            m.train_step_device(X, T, B, B, nf.LossKind.Mape, s)
        ctx.synchronize()
        t0 = time.perf_counter()
        for s in range(4, 4 + steps):
            m.train_step_device(X, T, B, B, nf.LossKind.Mape, s)
        ctx.synchronize()
        dt = (time.perf_counter() - t0) / steps
        out[["single", "dp_allreduce", "dp_levels"][exchange]] = {"ms_per_step": dt * 1e3,
                                                                   "variant": m.last_kernel_variant(0)}
        m.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
