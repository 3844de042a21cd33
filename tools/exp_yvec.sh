# A/B: float2 loads of Y / stores of dY in the MLP-only k_train path (product) vs scalar (tools/libnfg_prev.so); NeRF step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do for v in now prev; do
  L=paper_2201_05989_b200/libnfg.so; if [ $v = prev ]; then L=tools/libnfg_prev.so; fi
  echo "$v: $(NFG_LIB=$L python tools/nerf_time.py 2>&1 | tail -1)"
done; done
