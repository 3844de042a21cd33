# ncu evidence for the bench workload (one GPU). Usage: bash tools/gpu_ncu.sh <tag>
# Then, here (no GPU): python tools/ncu_summary.py <tag>
# Reports larger than ~20 MB (k_train with --import-source) are exported on the
# box to raw / details / source CSVs and deleted, so gpurun_out/ stays under
# the 64 MiB copy-back limit.
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out
# launch list of this library's kernels (mangled names start with _ZN3nfg)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:_ZN3nfg -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --infer-b 4194304 > gpurun_out/launches_$TAG.log 2>&1
for K in k_train k_adam k_infer; do
  timeout 600 ncu --set full --clock-control none --import-source on -k $K -s 3 -c 1 -o gpurun_out/prof_${K}_$TAG \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --infer-b 4194304 > gpurun_out/prof_${K}_$TAG.log 2>&1
  R=gpurun_out/prof_${K}_$TAG.ncu-rep
  if [ -f $R ]; then
    ncu -i $R --page raw --csv > gpurun_out/prof_${K}_${TAG}_raw.csv 2>/dev/null
    ncu -i $R --page details > gpurun_out/prof_${K}_${TAG}_details.txt 2>/dev/null
    if [ $(stat -c %s $R) -gt 20000000 ]; then
      ncu -i $R --page source --csv --print-source sass > gpurun_out/prof_${K}_${TAG}_source.csv 2>/dev/null
      gzip -9 gpurun_out/prof_${K}_${TAG}_source.csv
      rm -f $R
    fi
  fi
done
ls -la gpurun_out
# NeRF (config 4) launch list: steps 21-40 of a 40-step run
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 200 --csv \
    --log-file gpurun_out/nerf_launches_$TAG.csv python tools/nerf_prof.py 40 > gpurun_out/nerf_prof_$TAG.log 2>&1
du -sh gpurun_out
