cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_cfg3.json 2> gpurun_out/final_cfg3.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/final_cfg3.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline_sort']['frac'], d['roofline_build']['frac'], d['e2e']['ms_per_step'], d['clocks'], d.get('cpu_baseline',{}).get('value'))"
