cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/final_bench.json
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 2>&1 | tail -1 > gpurun_out/final_ref.json
python -c "
import json; d=json.load(open('gpurun_out/final_bench.json')); r=d['roofline']
print('value %.4g e2e %.4g pageable %.4g k_train %.1f adam %.1f infer %.4g frac %.3f infer_frac %.3f' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1e3, d['inference']['value'], r['frac'], d['roofline_infer']['frac']))
print('config1 %.4g giga %.4g nerf %.4g launches %d clocks %s' % (d['config1']['value'], d['gigapixel']['value'], d['nerf']['value'], d['gpu_launches'], d['clocks']))
e=json.load(open('gpurun_out/final_ref.json')); print('reference %.4g' % e['value'])"
