cd $GRAFT_REPO_ROOT
for i in $(seq 1 12); do
timeout 900 python -m pytest tests/test_gpu_headline.py -q --timeout 600 -k "test_headline_gradients and config1 and trained" --tb=line 2>&1 | grep -E "Error|assert|passed|failed" | head -4
done
