# Quick GPU check: selected GPU tests (pytest -k EXPR) + a short bench line.
# Usage: bash tools/gpu_quick.sh "<pytest -k expr>" [extra bench args]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${1:-smoke}
shift
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "$K" 2>&1 | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nerf "$@" 2>&1 | tail -3 > gpurun_out/quick_bench.json
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/quick_bench.json").read().strip().splitlines()[-1])
except Exception as e:
    print("bench failed", e, open("gpurun_out/quick_bench.json").read()[-2000:])
    raise SystemExit
r = d.get("roofline") or {}
print("value %.4g e2e %.4g pageable %.4g infer %.4g | k_train %.1f us frac %.3f | adam %.1f us | clocks %s" % (
    d["value"], d["e2e"]["value"], d.get("e2e_pageable", {}).get("value", 0), d["inference"]["value"],
    r.get("kernel_us", 0), r.get("frac", 0), d["phases_ms_per_step"]["adam"] * 1000, d["clocks"]))
PY
