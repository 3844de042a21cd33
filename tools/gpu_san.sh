cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $S --tool memcheck --error-exitcode 9 python tools/sanitize.py engines nerf more > gpurun_out/san_memcheck_r2f.log 2>&1; echo "memcheck rc $?"
timeout 1200 $S --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize.py engines > gpurun_out/san_racecheck_r2f.log 2>&1; echo "racecheck rc $?"
timeout 1200 $S --tool synccheck --error-exitcode 9 python tools/sanitize.py engines nerf > gpurun_out/san_synccheck_r2f.log 2>&1; echo "synccheck rc $?"
timeout 1200 $S --tool initcheck --error-exitcode 9 python tools/sanitize.py engines > gpurun_out/san_initcheck_r2f.log 2>&1; echo "initcheck rc $?"
for f in gpurun_out/san_*_r2f.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|engine|loss|Error|error" $f | head -8; done
