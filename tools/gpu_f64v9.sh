cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6
for v in 0 1; do BH_WALK_F64_V9=$v timeout 300 python bench.py --config cfg2 --precision fp64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/h.json 2>gpurun_out/h.err
python -c "
import json; d=json.loads(open('gpurun_out/h.json').read().strip().splitlines()[-1]); print('cfg2 fp64 v9d=$v', d['ms_per_step'], d['phase_ms_per_step']['walk'], d['roofline']['frac'], d['pp_per_step'], d['pc_per_step'])" || tail -5 gpurun_out/h.err
done
