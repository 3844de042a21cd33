cd $GRAFT_REPO_ROOT
for i in $(seq 1 10); do
timeout 900 python -m pytest tests/test_gpu_headline.py -q -s --timeout 600 -k "test_headline_gradients and trained and config1" 2>&1 | grep -oE "config1 [0-9]+ trained .*" | cut -c1-420
done
