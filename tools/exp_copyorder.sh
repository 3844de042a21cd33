# A/B: streamed copies enqueued right after the fused kernel (product) vs after the optimizer launches (tools/libnfg_prev.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do for v in now prev; do
  L=paper_2201_05989_b200/libnfg.so; if [ $v = prev ]; then L=tools/libnfg_prev.so; fi
  echo "$v: $(NFG_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 65536 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1))')"
done; done
