cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf 2>&1 | tail -1 > gpurun_out/t14.json
python -c "
import json; d=json.load(open('gpurun_out/t14.json')); r=d['roofline']
print('value %.4g e2e %.4g pageable %.4g k_train %.1f us' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us']))"
