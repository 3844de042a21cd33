cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in cur alias2 alias3 alias4; do echo "$v: $(KB_EVEN=1 ./tools/kbench_$v 262144 40 | head -1)"; done; done
