cd $GRAFT_REPO_ROOT
for f in "-DBH_MOM_TIMERS -DBH_BUCKET_DIAG=1" "-DBH_MOM_TIMERS -DBH_BUCKET_DIAG=2" "-DBH_MOM_TIMERS -DBH_BUCKET_DIAG=3"; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
echo "$f"; timeout 600 python tools/mom_timers.py cfg3 2>&1 | head -4
done
