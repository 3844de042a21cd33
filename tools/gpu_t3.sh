cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NFG_DEBUG_OCC=1 timeout 300 python tools/dbg/dbg_det_tc.py 2>&1 | grep -v "^\[nfg\]" | tail -6
for cfg in "1 2" "2 1" "2 2" "2 3" "2 4"; do
  set -- $cfg
  NFG_TRAIN_CTAS_PER_SM=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nerf --mlp-engine $1 --infer-b 1048576 2>/dev/null | tail -1 > gpurun_out/t3_$1_$2.json
  python -c "
import json; d=json.load(open('gpurun_out/t3_$1_$2.json')); r=d['roofline']
print('engine $1 ctas/SM $2: value %.4g  k_train %.1f us  adam %.1f us' % (d['value'], r['kernel_us'], d['phases_ms_per_step']['adam']*1000))"
done
