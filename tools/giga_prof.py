"""Gigapixel (config 3) training steps for a launch-list profile."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2201_05989_b200 import nf  # noqa: E402

print(bench.bench_gigapixel(nf, nf.default_context(), steps=6, warmup=3))
