cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in libnfg.so libnfg_mb4.so; do
  NFG_LIB=$GRAFT_REPO_ROOT/paper_2201_05989_b200/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-nerf --infer-b 1048576 2>&1 | tail -1 > gpurun_out/t11_$lib.json
  python -c "
import json; d=json.load(open('gpurun_out/t11_$lib.json')); r=d['roofline']
print('$lib: value %.4g e2e %.4g k_train %.1f us' % (d['value'], d['e2e']['value'], r['kernel_us']))"
done
