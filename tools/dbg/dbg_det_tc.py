"""Debug: run-to-run reproducibility of deterministic-mode steps per MLP engine."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
from paper_2201_05989_b200 import nf  # noqa: E402

g = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 16, features=2, n_min=16, n_max=1024)
for eng in (1, 2):
    for fp32 in (True, False):
        runs = []
        for _ in range(2):
            m = nf.FieldModel(options=nf.Options(table_fp32=fp32, deterministic=True, mlp_engine=eng))
            m.hash_cfg = g
            m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
            m.hyper = nf.AdamHyper(lr=1e-3)
            m.init(1337)
            rng = O.Pcg32(21, 4)
            X = rng.floats(20000 * 3).reshape(20000, 3)
            T = O.csg_sdf(X).reshape(-1, 1)
            l = m.gradients(X, T, nf.LossKind.Mape)
            runs.append((l, m.grads))
        (l0, g0), (l1, g1) = runs
        t = m.sizes[0]
        d = np.abs(g0 - g1)
        print(f"engine {eng} fp32 {fp32}: loss equal {l0 == l1}; grads differ at {np.count_nonzero(d)} entries "
              f"(tables {np.count_nonzero(d[:t])}, mlp {np.count_nonzero(d[t:])}), max {d.max():.3g}; "
              f"{m.last_kernel_variant(0)}", flush=True)
        if np.count_nonzero(d[t:]):
            idx = np.nonzero(d[t:])[0][:10]
            print("   first mlp diffs at", idx, g0[t:][idx], g1[t:][idx])
