"""Small fused train + inference + NeRF steps for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import oracle as O  # noqa: E402
from paper_2201_05989_b200 import nf  # noqa: E402

m = nf.FieldModel()
m.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512, dims=3)
m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
m.init(3)
rng = O.Pcg32(3, 3)
for step in range(1, 3):
    X = rng.floats(700 * 3).reshape(-1, 3)
    print("loss", m.train_step(X, O.csg_sdf(X).reshape(-1, 1), nf.LossKind.Mape, step))
print("eval", float(m.evaluate(X[:100]).sum()))
if "engines" in sys.argv:   # both tensor-core engines, several tiles per CTA (TMEM accumulators, rescale)
    for eng in (1, 2):
        e = nf.FieldModel(options=nf.Options(mlp_engine=eng))
        e.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << 14, features=2, n_min=16, n_max=512, dims=3)
        e.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
        e.init(4)
        X = rng.floats(70000 * 3).reshape(-1, 3)
        T = (O.csg_sdf(X).reshape(-1, 1) * np.linspace(0.01, 100.0, 70000, dtype=np.float32)[:, None])
        print("engine", eng, e.train_step(X, T.astype(np.float32), nf.LossKind.L2, 1),
              float(e.evaluate(X[:5000]).sum()), e.last_kernel_variant(0), e.last_kernel_variant(1))
if "nerf" in sys.argv:
    cams, focal = nf.orbit_cameras(2, width=16)
    imgs = nf.nerf_scene_render(cams, 16, 16, focal)
    nr = nf.NeRF(grid=nf.HashEncodingConfig(levels=16, table_size=1 << 12, features=2, n_min=16, n_max=128, dims=3),
                 target_samples=1 << 12, seed=1)
    nr.set_dataset(cams, imgs, 16, 16, focal)
    print("nerf", nr.train_step(1))
if "more" in sys.argv:
    d = nf.FieldModel(options=nf.Options(deterministic=True))
    d.hash_cfg = nf.HashEncodingConfig(levels=8, table_size=1 << 10, features=2, n_min=4, n_max=64, dims=2)
    d.mlp_cfg = nf.MlpConfig(hidden_layers=1, hidden_width=64, output_width=3,
                             output_activation=nf.OutputActivation.Sigmoid)
    d.init(1)
    X = rng.floats(300 * 2).reshape(-1, 2)
    print("det", d.train_step(X, np.full((300, 3), 0.5, np.float32), nf.LossKind.L2, 1))
    print("render", float(nf.render_image(d, 8, 8).sum()))
    t = nf.ImageTask(image=O.make_test_image(16, 16), width=16, height=16,
                     cfg=nf.HashEncodingConfig(levels=4, table_size=1 << 8, n_min=4, n_max=0),
                     batch_size=256, total_steps=3, log_interval=2)
    print("fit_image", [r.metric for r in nf.fit_image(t, 2).report.rows])
    img = nf.render_sdf_shaded(m, nf.Camera(), 8, 8)
    print("sdf render", float(img.sum()))
