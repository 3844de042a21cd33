cd $GRAFT_REPO_ROOT
for i in 1 2 3 4; do
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -q --timeout 600 --tb=line 2>&1 | grep -E "Error|assert|passed|failed" | cut -c1-600 | head -6
done
