cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/t10.json
python -c "
import json; d=json.load(open('gpurun_out/t10.json')); r=d['roofline']
print('value %.4g e2e %.4g pageable %.4g k_train %.1f us adam %.1f infer %.4g cpu %s' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1e3, d['inference']['value'], d['cpu_baseline']))"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 2>&1 | tail -1 > gpurun_out/t10_ref.json
python -c "
import json; d=json.load(open('gpurun_out/t10_ref.json')); print('reference', d['value'], d['cpu_baseline']['cores'], d['cpu_baseline']['phases_s_per_step'])"
