cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3
for p in 1 0 1 0; do
  if [ $p = 1 ]; then export NFG_NO_PDL=1; else unset NFG_NO_PDL; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/t19_$p.json
  python -c "
import json; d=json.load(open('gpurun_out/t19_$p.json')); r=d['roofline']
print('no_pdl=$p: value %.4g e2e %.4g ms/step %.4f k_train %.1f adam %.1f | config1 %.4g (%.4f ms) giga %.4g nerf %.4g' % (d['value'], d['e2e']['value'], d['ms_per_step'], r['kernel_us'], d['phases_ms_per_step']['adam']*1e3, d['config1']['value'], d['config1']['ms_per_step'], d['gigapixel']['value'], d['nerf']['value']))"
done
