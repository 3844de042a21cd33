cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --tb=short -p no:cacheprovider 2>&1 > gpurun_out/t27_$i.log
tail -1 gpurun_out/t27_$i.log
grep -nE "^E |FAILED" gpurun_out/t27_$i.log | cut -c1-400 | head -12
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf 2>&1 | tail -1 > gpurun_out/t27.json
python -c "
import json; d=json.load(open('gpurun_out/t27.json')); r=d['roofline']
print('value %.4g e2e %.4g k_train %.1f' % (d['value'], d['e2e']['value'], r['kernel_us']))"
