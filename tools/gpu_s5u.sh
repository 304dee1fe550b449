cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -k "sort or scan or order or keys or hilbert or schedule" 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh "" "-DBH_SORT_MATCH_TOP=0" "-DBH_SORT_UNIFORM=1"
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hilbert|k_sort_pass|k_sort_hist" --csv --log-file gpurun_out/h_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; grep -E "k_" gpurun_out/h_ll.csv | awk -F'","' '{print substr($5,1,40), $(NF)}' | tail -12
