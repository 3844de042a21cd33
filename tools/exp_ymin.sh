# A/B: CTAs per SM for the MLP-only k_train instantiations (NeRF colour network backward)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for v in base y3 y4; do if [ $v = base ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_$v.so; fi
echo "$v: $(NFG_LIB=$L python tools/nerf_time.py 2>&1 | tail -1)"; done; done
