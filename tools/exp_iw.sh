cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in base 20 28; do if [ $v = base ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_iw$v.so; fi
echo "iw=$v: $(NFG_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nerf | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["inference"])')"; done; done
