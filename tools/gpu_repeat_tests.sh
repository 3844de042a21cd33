# repeats the full GPU suite; keeps the logs of failing runs (flake hunting)
cd $GRAFT_REPO_ROOT
for i in $(seq 1 ${REPEATS:-3}); do
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --tb=long -rf -p no:cacheprovider > gpurun_out/rep_$i.log 2>&1
tail -1 gpurun_out/rep_$i.log
grep -nE "^E |FAILED" gpurun_out/rep_$i.log | cut -c1-600 | head -12
grep -q failed gpurun_out/rep_$i.log || rm -f gpurun_out/rep_$i.log
done
