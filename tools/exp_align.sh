# A/B: level row alignment of the device layout (2 = even rows, 8 = sector-aligned) for the lane-pair k_train
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do for a in 2 8; do echo "align $a: $(KB_ALIGN=$a ./tools/kbench_lp 262144 40 | head -1)"; done; done
