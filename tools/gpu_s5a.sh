cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s5_cfg3.json 2> gpurun_out/s5_cfg3.err; echo rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s5_cfg3.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','e2e','roofline','phase_ms_per_step','clocks','gpu_launches') if k in d})
for k in d:
    if k.startswith('roofline_') or k.startswith('e2e_'): print(k, d[k])
PY
