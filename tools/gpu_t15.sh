cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NFG_TRAIN_WS=1 timeout 600 python -m pytest tests/test_gpu_headline.py -q -x --timeout 600 -k "gradients" 2>&1 | tail -4
for ws in 0 1; do
  NFG_TRAIN_WS=$ws timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 1048576 2>&1 | tail -1 > gpurun_out/t15_$ws.json
  python -c "
import json; d=json.load(open('gpurun_out/t15_$ws.json')); r=d['roofline']
print('ws $ws: value %.4g e2e %.4g k_train %.1f us' % (d['value'], d['e2e']['value'], r['kernel_us']))"
done
cat /root/.nothing 2>/dev/null
