cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/infer_ab.py 16 98304 17 196608 261171 18 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['queries'], 'sync %.3g tc %.3g' % (d['sync_qps'], d['tc_qps']))
"
