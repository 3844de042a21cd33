"""In-kernel A/B of the inference MLP engine: fused k_infer (mma.sync) vs
k_infer_tc (tcgen05) at config 5 (3D L16 F2 T=2^19 + 32-64-64-1), same
parameters and queries, CUDA events on the library stream.
Usage: python tools/infer_ab.py [log2 queries ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_05989_b200 import nf  # noqa: E402


def main():
    # arguments: log2 sizes (<= 40) or explicit query counts
    sizes = [int(a) for a in sys.argv[1:]] or [16, 18, 20, 22, 24, 26]
    ctx = nf.Context(0)
    ms = {}
    for eng in (1, 2):
        m = nf.FieldModel(ctx, options=nf.Options(mlp_engine=eng))
        m.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, dims=3)
        m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
        m.init(1337)
        ms[eng] = m
    # random tables at the trained scale so the MLP sees realistic activations
    g = torch.Generator(device="cpu").manual_seed(1)
    P = ms[1].params
    nt = ms[1].sizes[0]
    P[:nt] = (torch.rand(nt, generator=g).numpy() - 0.5) * 0.2
    for m in ms.values():
        m.write(nf.BUF_PARAMS, P)
    stream = torch.cuda.ExternalStream(ctx.stream) if hasattr(ctx, "stream") else torch.cuda.current_stream()
    res = []
    gen = torch.Generator(device="cuda").manual_seed(7)
    for lg in sizes:
        n = 1 << lg if lg <= 40 else lg
        X = torch.rand(n, 3, device="cuda", generator=gen)
        outs = {}
        row = {"queries": n}
        for eng, m in ms.items():
            o = torch.empty(n, 1, device="cuda")
            for _ in range(3):
                m.evaluate_device(X, n, o)
            ctx.synchronize()
            reps = max(3, min(50, (1 << 24) // n))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                m.evaluate_device(X, n, o)
            e1.record(stream)
            ctx.synchronize()
            t = e0.elapsed_time(e1) / reps
            row["sync_ms" if eng == 1 else "tc_ms"] = t
            row["sync_qps" if eng == 1 else "tc_qps"] = n / t * 1e3
            row["variant_" + ("sync" if eng == 1 else "tc")] = m.last_kernel_variant(1)
            outs[eng] = o
        row["max_abs_diff"] = float((outs[1] - outs[2]).abs().max())
        row["max_abs_out"] = float(outs[1].abs().max())
        res.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
