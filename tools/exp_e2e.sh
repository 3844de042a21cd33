cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for cf in 0 1; do echo "copies_first=$cf: $(NFG_COPIES_FIRST=$cf python bench.py --steps 30 --warmup 5 --no-cpu-baseline --infer-b 1048576 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"])')"; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or invalid" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_train -c 12 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --infer-b 65536 > gpurun_out/ncu_e2e_check.log 2>&1; echo "ncu rc=$?"; grep -c "k_train" gpurun_out/ncu_e2e_check.log
