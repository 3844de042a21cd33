# A/B: lane pairs (product build) vs NFG_NO_LANE_PAIRS (tools/libnfg_nolp.so) through bench.py
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in lp nolp; do
  if [ $v = lp ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_$v.so; fi
  echo "$v: $(NFG_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1), round(d["inference"]["value"]/1e9,3), d["phases_ms_per_step"], (d.get("gigapixel") or {}).get("value"))')"
done; done
