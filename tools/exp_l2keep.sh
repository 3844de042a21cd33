# A/B: L2 evict_last hints for k_train's gathers/reductions (keep) and Adam's gradient loads (gkeep)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in base keep gkeep both; do
  if [ $v = base ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_$v.so; fi
  echo "$v: $(NFG_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 65536 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1), d["phases_ms_per_step"])')"
done; done
