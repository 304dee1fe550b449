cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_walk_schedules.py tests/test_gpu_walk_only.py tests/test_gpu_parity.py tests/test_gpu_decomposition.py -q -x 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg2" bash tools/walk_ab.sh "" ""
