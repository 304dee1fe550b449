cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02e
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02e/bench_cfg3.json 2> gpurun_out/r02e/bench_cfg3.err; echo cfg3 rc=$?
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/r02e/bench_cfg2.json 2> gpurun_out/r02e/bench_cfg2.err; echo cfg2 rc=$?
timeout 600 python bench.py --config cfg2 --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02e/bench_cfg2_fp64.json 2> gpurun_out/r02e/bench_cfg2_fp64.err; echo cfg2fp64 rc=$?
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02e/bench_cfg4.json 2> gpurun_out/r02e/bench_cfg4.err; echo cfg4 rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02e/bench_ref_cfg3.json 2> gpurun_out/r02e/bench_ref_cfg3.err; echo ref rc=$?
for c in cfg3 cfg4; do
python tools/step_cfg.py $c 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02e/ll_$c.csv python tools/step_cfg.py $c 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02e/ll_$c.csv gpurun_out/r02e/ll_$c.json "$c one step" | head -8
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02e/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("ms_per_step"), {k: round(v, 3) for k, v in d.get("phase_ms_per_step", {}).items()},
              (d.get("roofline") or {}).get("frac"), (d.get("roofline_sort") or {}).get("frac"),
              (d.get("roofline_build") or {}).get("frac"), (d.get("e2e") or {}).get("ms_per_step"),
              (d.get("e2e_plugin") or {}).get("ms_per_step"), d.get("value"), d.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
echo done
