cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 1 2; do echo "== engine $e"; KB_ENGINE=$e timeout 120 tools/kbench_pt 262144 20 2>&1 | head -10; done
