cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_nerf.py -q --timeout 600 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/t21.json
python -c "
import json; d=json.load(open('gpurun_out/t21.json')); print('nerf', d['nerf']['value'], d['nerf']['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'])"
