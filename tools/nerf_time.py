"""Config-4 NeRF step time only (bench.bench_nerf), for A/B builds via NFG_LIB."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2201_05989_b200 import nf  # noqa: E402

r = bench.bench_nerf(nf, nf.default_context(), steps=30, warmup=40)
print(round(r["ms_per_step"], 4), round(r["value"] / 1e6, 1))
