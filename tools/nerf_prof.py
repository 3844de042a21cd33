"""NeRF training steps for a launch-list profile (ncu --metrics gpu__time_duration.sum)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_05989_b200 import nf  # noqa: E402

W = 128
cams, focal = nf.orbit_cameras(16, width=W)
images = nf.nerf_scene_render(cams, W, W, focal)
nerf = nf.NeRF(lr=1e-2, target_samples=1 << 18, seed=1337)
nerf.set_dataset(cams, images, W, W, focal)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for s in range(1, n + 1):
    loss, nr, ns = nerf.train_step(s)
print("loss", loss, "rays", nr, "samples", ns)
