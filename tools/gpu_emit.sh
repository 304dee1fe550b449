cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh "-DBH_EMIT_WINDOW=0" ""
