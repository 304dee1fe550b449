cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_decomposition.py -q 2>&1 | tail -2
AB_CONFIGS="cfg3" bash tools/walk_ab.sh ""
