# A/B: in-kernel cooperative dW/db reduction (PG = 8 partials per item; tools/libnfg_pg32.so: 32) vs per-CTA float atomics (NFG_TRAIN_COOP=0)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in pg8 pg32 atomics; do
  L=paper_2201_05989_b200/libnfg.so; C=1
  if [ $v = pg32 ]; then L=tools/libnfg_pg32.so; fi
  if [ $v = atomics ]; then C=0; fi
  echo "$v: $(NFG_LIB=$L NFG_TRAIN_COOP=$C python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 65536 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1), d["phases_ms_per_step"])')"
done; done
