# tcgen05 engine checks + in-kernel inference A/B (one GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_width.py -q -x --timeout 600 2>&1 | tail -30
timeout 600 python tools/infer_ab.py 2>&1 | tail -12 | tee gpurun_out/infer_ab.log
