cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_walk_schedules.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "fp32 or scale or leaf or bucket or cfg or schedule" 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg2" bash tools/walk_ab.sh "-DBH_W9_PPSORT=0" "" "-DBH_W9_PPFLUSH=48"
