cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh "" "-DBH_SORT_VIDX=1" "-DBH_SORT_VIDX=1 -DBH_SORT_BLOCKS=4"
