cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider > gpurun_out/rep_$i.log 2>&1
tail -1 gpurun_out/rep_$i.log
grep -nE "^E |FAILED" gpurun_out/rep_$i.log | cut -c1-300 | head -8
done
