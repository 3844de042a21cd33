cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for srt in none 4 5 6; do for agg in 0 64 160 300; do
  if [ $srt = none ]; then R=$(KB_EVEN=1 KB_AGG=$agg ./tools/kbench_base 262144 30 | head -1); else R=$(KB_EVEN=1 KB_SORT=$srt KB_AGG=$agg ./tools/kbench_base 262144 30 | head -1); fi
  echo "sort=$srt agg=$agg: $R"
done; done
