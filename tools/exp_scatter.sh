cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in base skip5 skip8 skip16; do for srt in none 5; do
  if [ $srt = none ]; then KB_EVEN=1 ./tools/kbench_$v 262144 30 > gpurun_out/kb_${v}_$srt.log 2>&1; else KB_EVEN=1 KB_SORT=$srt ./tools/kbench_$v 262144 30 > gpurun_out/kb_${v}_$srt.log 2>&1; fi
  echo "== $v sort=$srt"; head -9 gpurun_out/kb_${v}_$srt.log
done; done
timeout 600 python -m pytest tests/test_gpu_shim.py -q -x 2>&1 | tail -3
