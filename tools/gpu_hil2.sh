cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg3" bash tools/walk_ab.sh "-DBH_HIL_CHUNK=2048" "" "-DBH_HIL_CHUNK=8192"
