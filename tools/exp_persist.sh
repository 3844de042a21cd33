# A/B: persisting-L2 access-policy window over the fp16 table shadow (1) or the gradient slab (2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in 0 1 2; do
  if [ $v = 0 ]; then unset NFG_L2_PERSIST; else export NFG_L2_PERSIST=$v; fi
  echo "persist $v: $(python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 65536 2>gpurun_out/persist_$v.err | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1), d["phases_ms_per_step"])')"
  head -2 gpurun_out/persist_$v.err
done; done
