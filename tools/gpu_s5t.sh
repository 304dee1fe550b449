cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -k "sort or scan or order or keys" 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg4 cfg2" bash tools/sort_ab.sh "" "-DBH_SORT_RANKASM=0"
