cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shim.py tests/test_gpu_tcgen05.py -q -x --timeout 600 2>&1 | tail -5
for e in 0 1; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nerf --mlp-engine $e 2>&1 | tail -1 > gpurun_out/t5_bench_$e.json
python -c "
import json; d=json.load(open('gpurun_out/t5_bench_$e.json')); r=d['roofline']
print('engine $e: value %.4g e2e %.4g pageable %.4g k_train %.1f us adam %.1f us' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1000))"
done
