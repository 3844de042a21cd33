cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r2a_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2a_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/r2a_bench.log 2>&1
bash tools/gpu_ncu.sh r2a > /dev/null 2>&1
tail -3 gpurun_out/r2a_tests.log; tail -1 gpurun_out/r2a_bench.log | cut -c1-600
