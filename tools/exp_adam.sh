cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for e in 0 1; do echo "eager=$e: $(NFG_ADAM_EAGER=$e python bench.py --steps 30 --warmup 5 --no-cpu-baseline --infer-b 1048576 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["phases_ms_per_step"], d["value"])')"; done; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
