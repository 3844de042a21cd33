# A/B after lane pairs: 2 CTAs/SM (255 regs) vs 3 CTAs/SM (168 regs, spills) for k_train
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in lp lp3; do echo "$v: $(KB_ALIGN=8 ./tools/kbench_$v 262144 40 | head -1)"; done; done
