cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NFG_DEBUG_OCC=1 timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -3
timeout 2000 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nerf 2>&1 | tail -1 > gpurun_out/t4_bench.json
python -c "
import json; d=json.load(open('gpurun_out/t4_bench.json')); r=d['roofline']
print('default: value %.4g e2e %.4g infer %.4g k_train %.1f us adam %.1f us' % (d['value'], d['e2e']['value'], d['inference']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1000))"
