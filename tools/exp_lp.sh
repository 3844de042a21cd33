# A/B: lane-pair gathers/reductions in k_train (tools/kbench_lp) vs one lane per (sample, level) (kbench_nolp)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do for v in lp nolp; do echo "$v: $(KB_ALIGN=${KB_ALIGN:-2} ./tools/kbench_$v 262144 40 | head -1)"; done; done
