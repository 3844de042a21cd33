# Round-end evidence on one box: GPU suite, smoke, bench (JSON), reference arm, ncu captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-final}
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
tail -1 gpurun_out/${TAG}_tests.log; grep -E "^E |FAILED" gpurun_out/${TAG}_tests.log | cut -c1-300 | head -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 400 gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; tail -c 300 gpurun_out/${TAG}_ref.json
if [ -n "$NCU" ]; then bash tools/gpu_ncu.sh $TAG > gpurun_out/${TAG}_ncu.log 2>&1; tail -2 gpurun_out/${TAG}_ncu.log; fi
