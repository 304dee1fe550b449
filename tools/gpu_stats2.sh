cd $GRAFT_REPO_ROOT
BH_NVCC_EXTRA="-DBH_W9_STATS" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
for c in cfg2 cfg3; do timeout 600 python tools/w9_stats.py $c 2>/dev/null > gpurun_out/w9stats_$c.json; done
BH_NVCC_EXTRA="" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1
python -c "
import json
for c in ('cfg2','cfg3'):
    d=json.load(open(f'gpurun_out/w9stats_{c}.json')); print(c, {k:(round(v,3) if isinstance(v,float) else v) for k,v in d.items() if k!='peak_frontier_hist_by10'})
"
