cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nerf 2>&1 | tail -1 > gpurun_out/t1_bench.json
python - <<'PY'
import json
d = json.loads(open("gpurun_out/t1_bench.json").read())
r = d.get("roofline") or {}
print("value %.4g e2e %.4g infer %.4g | k_train %.1f us | adam %.1f us" % (d["value"], d["e2e"]["value"], d["inference"]["value"], r.get("kernel_us", 0), d["phases_ms_per_step"]["adam"] * 1000))
PY
