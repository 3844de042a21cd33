cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 2>&1 | tail -3
for p in 1 0; do
 for rep in 1 2; do
  if [ $p = 1 ]; then export NFG_NO_PDL=1; else unset NFG_NO_PDL; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 1048576 2>&1 | tail -1 > gpurun_out/t16_$p.json
  python -c "
import json; d=json.load(open('gpurun_out/t16_$p.json')); r=d['roofline']
print('no_pdl=$p: value %.4g e2e %.4g k_train %.1f us adam %.1f us ms/step %.4f' % (d['value'], d['e2e']['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1e3, d['ms_per_step']))"
 done
done
