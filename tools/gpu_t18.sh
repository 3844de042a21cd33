cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/t18.json
python -c "
import json; d=json.load(open('gpurun_out/t18.json')); r=d['roofline']
print('value %.4g e2e %.4g pageable %.4g k_train %.1f us adam %.1f infer %.4g frac %.3f' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1e3, d['inference']['value'], r['frac']))
print('config1', d['config1']); print('giga', d['gigapixel']['value'], 'nerf', d['nerf']['value']); print('cpu', d['cpu_baseline']['value'], d['cpu_baseline'].get('inference_queries_per_s'))"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 2>&1 | tail -1 > gpurun_out/t18_ref.json
python -c "
import json; d=json.load(open('gpurun_out/t18_ref.json')); print('reference', d['value'], d['cpu_baseline'])"
