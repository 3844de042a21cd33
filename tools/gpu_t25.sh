cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider 2>&1 > gpurun_out/t25_$i.log
tail -2 gpurun_out/t25_$i.log
grep -nE "^E |FAILED" gpurun_out/t25_$i.log | cut -c1-400 | head -12
done
