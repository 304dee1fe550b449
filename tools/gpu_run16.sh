cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
AB_CONFIGS="cfg3 cfg2" bash tools/walk_ab.sh "" "-DBH_W9_PPFLUSH=56" "-DBH_W9_PPFLUSH=64 -DBH_W9_FLUSH=20"
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_cfg3.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/ll_cfg3.csv gpurun_out/ll_cfg3.json "cfg3 one step" | head -14
echo done
