cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_abi.py tests/test_harness.py tests/test_gpu_integration_doc.py tests/test_gpu_parity.py -q -x -k "not golden_tolerance" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pl.json 2>gpurun_out/pl.err; python -c "
import json; d=json.loads(open('gpurun_out/pl.json').read().strip().splitlines()[-1]); print('plugin ms', d['e2e_plugin']['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'step', d['ms_per_step'])" || tail -5 gpurun_out/pl.err
