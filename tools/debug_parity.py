"""Diagnostics for GPU-vs-oracle parity (prints error magnitudes)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np
import oracle as O
from paper_2201_05989_b200 import nf

def model(grid, hidden=2, n_out=1, sig=False, fp32=True, fused=True, lr=1e-3):
    m = nf.FieldModel(options=nf.Options(table_fp32=fp32, fused_train=fused))
    m.hash_cfg = grid
    m.mlp_cfg = nf.MlpConfig(hidden_layers=hidden, hidden_width=64, output_width=n_out,
                             output_activation=nf.OutputActivation.Sigmoid if sig else nf.OutputActivation.Linear)
    m.hyper = nf.AdamHyper(lr=lr)
    m.init(1337)
    return m

g = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 12, features=2, n_min=16, n_max=256)
for hidden, n_out, sig in [(2, 1, False), (2, 3, True), (1, 4, False)]:
    m = model(g, hidden, n_out, sig)
    mc = O.MlpCfg(32, hidden, 64, n_out, sig)
    t, w, b = m.sizes
    P = m.params
    W, bb = P[t:t + w], P[t + w:]
    rng = np.random.default_rng(0)
    Y = rng.uniform(-1, 1, (1000, 32)).astype(np.float32)
    out = m.mlp_forward(Y)
    ref = O.mlp_forward(mc, W, bb, Y)
    print("fwd", hidden, n_out, sig, "maxdiff", np.abs(out - ref).max(), "maxref", np.abs(ref).max(),
          "out[:2]", out[:2].ravel()[:4], "ref[:2]", ref[:2].ravel()[:4])
    dOut = (rng.uniform(-1, 1, (1000, n_out)) * 1e-5).astype(np.float32)
    dY = m.mlp_backward(Y, dOut)
    _, gW, gbb, dYo = O.mlp_forward_backward(mc, W, bb, Y, dOut)
    G = m.grads
    for name, a, r in (("gW", G[t:t + w], gW), ("gb", G[t + w:], gbb), ("dY", dY, dYo)):
        print("  bwd", name, "rel", np.linalg.norm(a - r) / np.linalg.norm(r), "norms", np.linalg.norm(a), np.linalg.norm(r))

# train step parity
for fused in (True, False):
    g = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512)
    m = model(g, fused=fused)
    f = O.Field(O.GridCfg(levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512, dims=3),
                O.MlpCfg(hidden_layers=2, hidden_width=64, output_width=1), O.Hyper(lr=1e-3))
    f.init(1337)
    print("init equal", np.array_equal(m.params, f.params))
    rng = O.Pcg32(21, 4)
    for step in range(1, 4):
        X = rng.floats(3000 * 3).reshape(3000, 3)
        T = rng.floats(3000).reshape(3000, 1) * 0.6 - 0.3
        lg = m.train_step(X, T, 1, step)
        lo = f.train_step(X, T, 1, step)
        d = np.abs(m.params - f.params)
        print("fused" if fused else "staged", "step", step, "loss", lg, lo, "param maxdiff", d.max(),
              "frac>1e-4", np.mean(d > 1e-4), "tab", d[:m.sizes[0]].max(), "W", d[m.sizes[0]:].max())

# gradient parity (no Adam)
g = nf.HashEncodingConfig(dims=3, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512)
for kind in (0, 1, 2):
    m = model(g)
    P = m.params
    t, w, b = m.sizes
    rng = O.Pcg32(21, 4)
    X = rng.floats(3000 * 3).reshape(3000, 3)
    T = rng.floats(3000).reshape(3000, 1) * 0.6 - 0.3
    lg = m.gradients(X, T, kind)
    G = m.grads
    og = O.GridCfg(levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512, dims=3)
    mc = O.MlpCfg(32, 2, 64, 1, False)
    Y, cache = O.encode_forward(og, P[:t], X)
    pred = O.mlp_forward(mc, P[t:t + w], P[t + w:], Y)
    lo, dp = O.loss_with_grad(kind, pred, T)
    _, gW, gb, dY = O.mlp_forward_backward(mc, P[t:t + w], P[t + w:], Y, dp)
    gt = np.zeros(t, np.float32)
    O.encode_backward(og, cache, dY, gt)
    print("grad kind", kind, "loss", lg, lo)
    for name, a, r in (("tab", G[:t], gt), ("W", G[t:t + w], gW), ("b", G[t + w:], gb)):
        print("   ", name, "rel", np.linalg.norm(a - r) / np.linalg.norm(r), "sign agree(|r|>1e-3max)",
              np.mean(np.sign(a[np.abs(r) > 1e-3 * np.abs(r).max()]) == np.sign(r[np.abs(r) > 1e-3 * np.abs(r).max()])))

# image trajectory
from _tasks import fit_image
w = h = 128
rgb = O.make_test_image(w, h)
g = nf.HashEncodingConfig(dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=64)
m = model(g, n_out=3, sig=True, lr=1e-2)
m.schedule = nf.default_schedule(300)
f = O.Field(O.GridCfg(levels=16, table_size=1 << 14, features=2, n_min=16, n_max=64, dims=2),
            O.MlpCfg(hidden_layers=2, hidden_width=64, output_width=3, sigmoid=True), O.Hyper(lr=1e-2))
f.init(1337)
f.set_schedule(O.default_milestones(300))
rg = fit_image(m, rgb, w, h, seed=1337, batch=1 << 12, total_steps=300, log_interval=25)
ro = fit_image(f, rgb, w, h, seed=1337, batch=1 << 12, total_steps=300, log_interval=25)
for a, b in zip(rg, ro):
    print("img", a, b)
