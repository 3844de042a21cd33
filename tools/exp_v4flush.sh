# A/B: dW flush with 16-byte vector reductions after a warp transpose (product) vs scalar atomics (tools/libnfg_nov4.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in v4 nov4; do
  L=paper_2201_05989_b200/libnfg.so; if [ $v = nov4 ]; then L=tools/libnfg_nov4.so; fi
  echo "$v: $(NFG_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 65536 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), round(d["e2e"]["value"]/1e6,1), d["phases_ms_per_step"])')"
done; done
