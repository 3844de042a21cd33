"""e2e train_step on pageable numpy arrays vs pinned buffers at config 2
(B = 2^18), for NFG_COPY_THREADS in the environment. Prints samples/s."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_05989_b200 import nf  # noqa: E402

B = 1 << 18
ctx = nf.Context(0)
m = nf.FieldModel(ctx)
m.hash_cfg = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)
m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
m.hyper = nf.AdamHyper(lr=1e-4)
m.init(1337)
rng = np.random.default_rng(1)
X = rng.random((B, 3), dtype=np.float32)
T = rng.random((B, 1), dtype=np.float32)
Xh, Th = nf.PinnedBuffer((B, 3)), nf.PinnedBuffer((B, 1))
Xh.array[:] = X
Th.array[:] = T
t0 = time.perf_counter()
for _ in range(20):
    Xh.array[:] = X
dt = (time.perf_counter() - t0) / 20
print(f"numpy pageable->pinned copy of X: {X.nbytes / dt / 1e9:.1f} GB/s (1 thread)")
step = 0


def run(xp, tp, n=20):
    global step
    for _ in range(3):
        step += 1
        m.train_step_host_ptr(xp, tp, B, nf.LossKind.Mape, step)
    t0 = time.perf_counter()
    for _ in range(n):
        step += 1
        m.train_step_host_ptr(xp, tp, B, nf.LossKind.Mape, step)
    return B * n / (time.perf_counter() - t0)


print(f"threads={os.environ.get('NFG_COPY_THREADS', 'default')} cpus={os.cpu_count()} "
      f"pinned {run(Xh.ptr, Th.ptr):.3e} pageable {run(X.ctypes.data, T.ctypes.data):.3e} samples/s")
