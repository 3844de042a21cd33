"""Wall-clock cost of one synchronous host-pointer train_step (pinned buffers) at several batch sizes."""
import time, numpy as np, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2201_05989_b200 import nf
m = nf.FieldModel()
m.hash_cfg = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)
m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
m.init(1)
for B in (1 << 10, 1 << 14, 1 << 18):
    Xh = nf.PinnedBuffer((B, 3)); Th = nf.PinnedBuffer((B, 1))
    Xh.array[:] = np.random.rand(B, 3); Th.array[:] = np.random.rand(B, 1)
    for i in range(5): m.train_step_host_ptr(Xh.ptr, Th.ptr, B, nf.LossKind.Mape, i + 1)
    t0 = time.perf_counter(); n = 50
    for i in range(n): m.train_step_host_ptr(Xh.ptr, Th.ptr, B, nf.LossKind.Mape, 10 + i)
    dt = (time.perf_counter() - t0) / n
    print(f"B={B}: {dt*1e6:.1f} us per synchronous train_step")
    Xh.free(); Th.free()
