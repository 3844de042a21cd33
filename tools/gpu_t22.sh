cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_headline.py -q --timeout 600 -k "test_headline_gradients and config1 and trained" 2>&1 | grep -E "AssertionError|assert|passed|failed|report" | head -8
done
