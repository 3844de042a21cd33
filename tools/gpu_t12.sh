cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -4
