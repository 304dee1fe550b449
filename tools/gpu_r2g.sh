cd $GRAFT_REPO_ROOT
# spill path exercised: shared frontier of 96 entries spills above 64
BH_NVCC_EXTRA="-DBH_W9_FCAP=96 -DBH_W9_CHECK=1" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_walk_schedules.py tests/test_gpu_scale.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32" 2>&1 | tail -3
AB_CONFIGS="cfg3" bash tools/walk_ab.sh "" "-DBH_W9_MINB=7" "-DBH_W9_FCAP=96 -DBH_W9_MINB=7" "-DBH_W9_MINB=7 -DBH_W9_FLUSH=24"
