cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg3 cfg2" bash tools/walk_ab.sh "" "-DBH_W9_PPPREF=0"
