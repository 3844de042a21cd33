# A/B: Adam eager (p/m/v loaded with g) vs lazy (g first) on config 3 (sparse gradients)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in default 1 0; do
  if [ $v = default ]; then unset NFG_ADAM_EAGER; else export NFG_ADAM_EAGER=$v; fi
  echo "eager=$v: $(python bench.py --steps 10 --warmup 3 --no-cpu-baseline --infer-b 65536 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["phases_ms_per_step"], d["gigapixel"]["ms_per_step"])')"
done; done
