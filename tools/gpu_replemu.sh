cd $GRAFT_REPO_ROOT
for c in cfg3 cfg2; do timeout 900 python tools/repl_emulate.py $c 2,4,8 > gpurun_out/repl_emu_$c.json 2> gpurun_out/repl_emu.err; echo "$c rc=$?"; tail -2 gpurun_out/repl_emu.err; python -c "
import json; d=json.load(open('gpurun_out/repl_emu_$c.json')); print(d['single_gpu_step_ms'], {R:(v['per_rank_device_ms'], v['device_efficiency_upper_bound'], v['walk_max_over_mean']) for R,v in d['ranks'].items()})"; done
