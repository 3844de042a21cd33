import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2201_05989_b200 import nf
B = 1 << 18
X = torch.rand(B, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
c = X - 0.5
T = (torch.sqrt((c * c).sum(1)) - 0.3).unsqueeze(1).contiguous()
for det in (False, True):
    ctx = nf.Context(0)
    m = nf.FieldModel(ctx, options=nf.Options(deterministic=det))
    m.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, dims=3)
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
    m.init(1)
    for s in range(1, 4): m.train_step_device(X, T, B, B, nf.LossKind.Mape, s)
    ctx.synchronize()
    ctx.lib.nfg_ctx_set_profiling(ctx.h, 1)
    import ctypes as C
    ms = (C.c_double * 4)(); n = C.c_int64()
    ctx.lib.nfg_ctx_read_profile(ctx.h, ms, C.byref(n))
    t0 = time.perf_counter()
    for s in range(4, 14): m.train_step_device(X, T, B, B, nf.LossKind.Mape, s)
    ctx.synchronize()
    dt = (time.perf_counter() - t0) / 10
    ctx.lib.nfg_ctx_read_profile(ctx.h, ms, C.byref(n))
    print("det" if det else "default", "%.3f ms/step" % (dt * 1e3), "phases ms", [round(ms[i] / 10, 3) for i in range(4)])
