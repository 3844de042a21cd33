# A/B: 32-byte sector gathers (product build) vs 8-byte pair loads (tools/libnfg_nosector.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in sector nosector g16; do   # variants built with EXTRA=-DNFG_NO_SECTOR_LOADS / -DNFG_GATHER16 (removed after the experiment)
  if [ $v = sector ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_$v.so; fi
  echo "$v: $(NFG_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nerf | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["inference"], d["value"])')"
done; done
