cd $GRAFT_REPO_ROOT
BH_NVCC_EXTRA="-DBH_MOM_TIMERS" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
timeout 600 python tools/mom_timers.py cfg3 2>&1 | head -4
