cd $GRAFT_REPO_ROOT
for i in $(seq 1 40); do
  timeout 300 python -m pytest "tests/test_gpu_headline.py::test_headline_gradients[config1-True-trained]" "tests/test_gpu_headline.py::test_headline_gradients[config1-False-trained]" -q --timeout 300 --tb=short -p no:cacheprovider > gpurun_out/flake.log 2>&1
  if ! grep -q "2 passed" gpurun_out/flake.log; then echo "run $i FAILED"; grep -E "^E " gpurun_out/flake.log | cut -c1-1500 | head -12; fi
done
echo done
