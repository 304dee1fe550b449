cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh ""
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_emit|k_mom_lists" --csv --log-file gpurun_out/e_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; grep -E "k_" gpurun_out/e_ll.csv | awk -F'","' '{print substr($5,1,30), $(NF)}' | tail -3
