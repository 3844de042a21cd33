cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in alias tw8 tw2x3; do echo "$v: $(KB_EVEN=1 ./tools/kbench_$v 262144 40 | head -1)"; done; done
