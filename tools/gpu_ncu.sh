cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline --infer-b 4194304 > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_train -s 2 -c 1 -o gpurun_out/prof_train python bench.py --steps 2 --warmup 2 --no-cpu-baseline --infer-b 1048576 > gpurun_out/prof_train.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_adam -s 4 -c 1 -o gpurun_out/prof_adam python bench.py --steps 2 --warmup 2 --no-cpu-baseline --infer-b 1048576 > gpurun_out/prof_adam.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_infer -s 2 -c 1 -o gpurun_out/prof_infer python bench.py --steps 2 --warmup 2 --no-cpu-baseline --infer-b 4194304 > gpurun_out/prof_infer.log 2>&1
ls -la gpurun_out
