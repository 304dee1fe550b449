cd $GRAFT_REPO_ROOT
for f in "-DBH_MOM_TIMERS" "-DBH_MOM_TIMERS -DBH_BUCKET_ONEPASS=0" "-DBH_MOM_TIMERS -DBH_MOM_MINB=2"; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
for c in cfg3; do echo "$c $f"; timeout 600 python tools/mom_timers.py $c 2>&1 | head -4; done
done
