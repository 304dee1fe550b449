cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_walk_only.py -q 2>&1 | tail -5
