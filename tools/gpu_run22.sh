cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in cfg3 cfg4; do
python tools/step_cfg.py $c 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_$c.csv python tools/step_cfg.py $c 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/ll_$c.csv gpurun_out/ll_$c.json "$c one step" | head -14
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2>gpurun_out/b3.err; python -c "
import json; d=json.loads(open('gpurun_out/b3.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms_per_step'], d['roofline']['frac'], d['roofline_build'], d['roofline_sort']['frac'], d['e2e_plugin'])"
echo done
