cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_decomposition.py tests/test_abi.py -q 2>&1 | tail -2
timeout 1500 python tools/dist_host.py cfg3 1 5 --replicated > gpurun_out/repl_host_cfg3.json 2> gpurun_out/repl_host.err; echo rc=$?; tail -2 gpurun_out/repl_host.err
python -c "
import json; d=json.load(open('gpurun_out/repl_host_cfg3.json'))
for R,v in d['ranks'].items(): print(R, 'wall', v['wall_ms'], 'dev_sum', v['device_ms_sum'], 'host_exposed', v['host_exposed_ms'])
"
bash tools/mrank_smoke.sh 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline --decomp replicated > gpurun_out/mr_r.json 2> gpurun_out/mr_r.err; echo "mrank rc=$?"; tail -c 200 gpurun_out/mr_r.json
