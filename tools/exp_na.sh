# A/B: k_infer hashed-level gathers with L1::no_allocate (tools/libnfg_na.so) vs the product build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in base na; do if [ $v = base ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_$v.so; fi
echo "$v: $(NFG_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nerf | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["inference"]["value"]/1e9,3), round(d["value"]/1e6,1))')"; done; done
