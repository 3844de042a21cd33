cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NFG_DEBUG_OCC=1 timeout 300 python tools/dbg/dbg_det_tc.py 2>&1 | tail -20
