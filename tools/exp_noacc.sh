cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in base2 noacc2 noacc3; do echo "$v: $(KB_EVEN=1 ./tools/kbench_$v 262144 40 | head -1)"; done; done
