set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -60
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 2>&1 | tail -5
