cd $GRAFT_REPO_ROOT
for r in 1 2 3; do for v in ts ws; do echo "$v: $(KB_EVEN=1 ./tools/kbench_$v 262144 40 | head -1)"; done; done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 1048576 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["phases_ms_per_step"])'
