cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do for v in nopair pair; do echo "$v: $(KB_EVEN=1 ./tools/kbench_$v 262144 40 | head -1)"; done; done
KB_EVEN=1 ./tools/kbench_pair 262144 40
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
