cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err; echo rc=$?
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err; echo rc=$?
python -c "
import json
for f in ['gpurun_out/b2.json','gpurun_out/b3.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['phase_ms_per_step'], d['roofline_sort'])
    except Exception as e: print(f, e)
"
