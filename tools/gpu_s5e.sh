cd $GRAFT_REPO_ROOT
for f in "-DBH_W9_STATS" "-DBH_W9_STATS -DBH_W9_HALVES=0"; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
echo "[$f]"
timeout 600 python tools/w9_stats.py cfg3 2>&1 | tail -40 | tr -d '\n' ; echo
done
