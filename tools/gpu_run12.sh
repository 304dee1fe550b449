cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg2 cfg3" bash tools/walk_ab.sh "-DBH_W9_PPPACK=0" ""
timeout 1500 python -m pytest tests/test_gpu_walk_schedules.py tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
echo done
