cd $GRAFT_REPO_ROOT
BH_NVCC_EXTRA="-DBH_W9_STATS" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
for c in cfg2 cfg3 cfg4; do timeout 600 python tools/w9_stats.py $c 2>&1 | tail -40 > gpurun_out/w9stats_$c.json; done
cat gpurun_out/w9stats_*.json
