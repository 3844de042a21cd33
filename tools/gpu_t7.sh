cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NFG_DEBUG_OCC=1 timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_tcgen05.py tests/test_gpu_deterministic.py tests/test_gpu_dp.py tests/test_gpu_width.py -q -x --timeout 600 2>&1 | tail -5
for lib in libnfg.so libnfg_g1.so; do
 for e in 0 1; do
  NFG_LIB=$GRAFT_REPO_ROOT/paper_2201_05989_b200/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --mlp-engine $e --infer-b 1048576 2>&1 | tail -1 > gpurun_out/t7_${lib}_$e.json
  python -c "
import json; d=json.load(open('gpurun_out/t7_${lib}_$e.json')); r=d['roofline']
print('$lib engine $e: value %.4g e2e %.4g pageable %.4g k_train %.1f us adam %.1f us' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1000))"
 done
done
