cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=8 2>&1 | tail -16
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_sort" --clock-control none --csv --log-file gpurun_out/sl3_hist.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
python tools/sort_ll.py gpurun_out/sl3_hist.csv | head -4
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/b3_default.json 2> gpurun_out/b3_default.err; echo rc=$?
timeout 900 python bench.py --config cfg2 --precision fp64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b2_fp64.json 2> gpurun_out/b2_fp64.err; echo rc=$?
tail -c 3000 gpurun_out/b3_default.json; echo; tail -c 2500 gpurun_out/b2_fp64.json; tail -5 gpurun_out/b2_fp64.err
echo done
