cd $GRAFT_REPO_ROOT
for r in 1 2; do for cv in none 100 75 60 50; do if [ $cv = none ]; then echo "default: $(KB_EVEN=1 ./tools/kbench_alias 262144 40 | head -1)"; else echo "carve=$cv: $(NFG_TRAIN_CARVEOUT=$cv KB_EVEN=1 ./tools/kbench_alias 262144 40 | head -1)"; fi; done; done
