cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_walk_schedules.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "fp32 or scale or leaf or bucket or cfg or schedule" 2>&1 | tail -2
for c in cfg3 cfg2; do
for hv in 0 1; do BH_WALK_HILBERT=$hv timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/h.json 2>gpurun_out/h.err
python -c "
import json; d=json.loads(open('gpurun_out/h.json').read().strip().splitlines()[-1]); print('$c hilbert=$hv', d['ms_per_step'], d['phase_ms_per_step']['walk'], d['roofline']['frac'])" || tail -5 gpurun_out/h.err
done; done
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hilbert|k_walk9" --csv --log-file gpurun_out/hil_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; grep -E "k_hilbert|k_walk9" gpurun_out/hil_ll.csv | awk -F'","' '{print $5, $(NF)}' | tail -4
