cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg3 cfg2 cfg4" bash tools/walk_ab.sh "" "-DBH_W9_PPFLUSH=96" "-DBH_W9_PPFLUSH=128"
