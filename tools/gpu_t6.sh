cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x --timeout 600 2>&1 | tail -15
timeout 300 python tools/dp_levels_prof.py 20 2>&1 | tail -2
DP_ONLY=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/dp_levels_launches.csv python tools/dp_levels_prof.py 3 > /dev/null 2>&1
DP_ONLY=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/dp_single_launches.csv python tools/dp_levels_prof.py 3 > /dev/null 2>&1
ls gpurun_out | grep dp_
