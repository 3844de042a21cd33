# A/B: first streamed chunk = one wave of tiles (num_sms x 128 samples, default) vs 4096 / 8192 (NFG_STREAM_CHUNK0)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do for v in 0 4096 8192; do
  if [ $v = 0 ]; then unset NFG_STREAM_CHUNK0; else export NFG_STREAM_CHUNK0=$v; fi
  echo "chunk0=$v: $(python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 65536 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1))')"
done; done
