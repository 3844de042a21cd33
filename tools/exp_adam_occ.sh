# A/B: CTAs per SM of the grid-stride Adam loop (NFG_ADAM_GRID; 5 are resident at 48 registers)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in 5 8 12 16 32 64; do
  echo "grid $v/SM: $(NFG_ADAM_GRID=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["phases_ms_per_step"], d["roofline_adam"]["achieved"])')"
done; done
