cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 tools/tc_probe 2>&1 | tee gpurun_out/tc_probe.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_infer_tc -s 2 -c 1 -o gpurun_out/prof_k_infer_tc_r2 python tools/infer_ab.py 22 > gpurun_out/prof_k_infer_tc_r2.log 2>&1
tail -3 gpurun_out/prof_k_infer_tc_r2.log
