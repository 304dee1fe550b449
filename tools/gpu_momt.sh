cd $GRAFT_REPO_ROOT
BH_NVCC_EXTRA="-DBH_MOM_TIMERS" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
for c in cfg3 cfg4; do echo $c; timeout 600 python tools/mom_timers.py $c 2>&1 | tail -30; done
