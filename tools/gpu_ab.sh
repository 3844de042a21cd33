# A/B of two library builds on one box: bench.py alternating NFG_LIB, then the GPU suite on the default build.
#   AB_LIBS="paper_2201_05989_b200/libnfg_base.so paper_2201_05989_b200/libnfg.so" bash tools/gpu_ab.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LIBS=${AB_LIBS:-"paper_2201_05989_b200/libnfg_base.so paper_2201_05989_b200/libnfg.so"}
for r in $(seq 1 ${AB_REPS:-3}); do
  for lib in $LIBS; do
    tag=$(basename $lib .so)
    NFG_LIB=$PWD/$lib timeout 600 python bench.py --steps ${AB_STEPS:-50} --warmup 5 ${AB_ARGS} > gpurun_out/ab_${tag}_$r.json 2> gpurun_out/ab_${tag}_$r.err
    python - gpurun_out/ab_${tag}_$r.json $tag <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]; ri = d.get("roofline_infer", {})
print(f"{sys.argv[2]:14s} value {d['value']:.4g} e2e {d['e2e']['value']:.4g} k_train_us {r['kernel_us']:.1f} frac {r['frac']:.3f} "
      f"infer {d['inference']['value'] if isinstance(d.get('inference'), dict) and 'value' in d['inference'] else '-'} "
      f"k_infer_us {ri.get('kernel_us', 0):.1f} ms/step {d['ms_per_step']:.4f} clk {d['clocks']['sm_mhz']}")
PY
  done
done
if [ -n "$AB_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1
  tail -1 gpurun_out/ab_tests.log; grep -E "^E |FAILED" gpurun_out/ab_tests.log | cut -c1-400 | head -10
fi
