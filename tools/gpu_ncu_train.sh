# k_train only: ncu --set full with source correlation exported per CUDA line and per SASS line.
#   bash tools/gpu_ncu_train.sh <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k k_train -s 3 -c 1 -o gpurun_out/prof_k_train_$TAG \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --infer-b 4194304 > gpurun_out/prof_k_train_$TAG.log 2>&1
R=gpurun_out/prof_k_train_$TAG.ncu-rep
ncu -i $R --page details > gpurun_out/prof_k_train_${TAG}_details.txt 2>/dev/null
ncu -i $R --page raw --csv > gpurun_out/prof_k_train_${TAG}_raw.csv 2>/dev/null
ncu -i $R --page source --csv --print-source cuda > gpurun_out/prof_k_train_${TAG}_cuda.csv 2>/dev/null
ncu -i $R --page source --csv --print-source sass > gpurun_out/prof_k_train_${TAG}_source.csv 2>/dev/null
gzip -9 -f gpurun_out/prof_k_train_${TAG}_cuda.csv gpurun_out/prof_k_train_${TAG}_source.csv
rm -f $R
ls -la gpurun_out | grep $TAG
