cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_tcgen05.py -q --timeout 600 -k "other_feature" 2>&1 | tail -15
