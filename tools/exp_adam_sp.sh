# A/B: quads per thread on sparse Adam steps (NFG_ADAM_QUAD_GROUP: product 2, tools/libnfg_qg{1,4}.so) on config 3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in qg1 qg4; do NFG_LIB=tools/libnfg_$v.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k adam 2>&1 | tail -1; done
for r in 1 2; do for v in qg2 qg1 qg4; do if [ $v = qg2 ]; then L=paper_2201_05989_b200/libnfg.so; else L=tools/libnfg_$v.so; fi
echo "$v: $(NFG_LIB=$L python tools/giga_prof.py 2>&1 | tail -1 | python -c 'import ast,sys; d=ast.literal_eval(sys.stdin.read()); print(round(d["ms_per_step"],4), d["phases_ms_per_step"])')"; done; done
