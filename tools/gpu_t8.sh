cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x --timeout 600 2>&1 | tail -4
for c0 in 0 9472 18944 56832; do
  NFG_STREAM_CHUNK0=$c0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 1048576 2>&1 | tail -1 > gpurun_out/t8_$c0.json
  python -c "
import json; d=json.load(open('gpurun_out/t8_$c0.json')); r=d['roofline']
print('chunk0 $c0: value %.4g e2e %.4g pageable %.4g k_train %.1f us' % (d['value'], d['e2e']['value'], d['e2e_pageable']['value'], r['kernel_us']))"
done
