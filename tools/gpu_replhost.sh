cd $GRAFT_REPO_ROOT
timeout 1500 python tools/dist_host.py cfg3 1,2,8 5 --replicated > gpurun_out/repl_host_cfg3.json 2> gpurun_out/repl_host.err; echo rc=$?; tail -3 gpurun_out/repl_host.err
python -c "
import json; d=json.load(open('gpurun_out/repl_host_cfg3.json'))
for R,v in d['ranks'].items(): print(R, 'wall', v['wall_ms'], 'dev_sum', v['device_ms_sum'], 'host_exposed', v['host_exposed_ms'], [ (x['wall_ms'], x['device_ms'], x['phases']) for x in v['per_rank']][:1])
"
