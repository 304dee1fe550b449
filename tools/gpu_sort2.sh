cd $GRAFT_REPO_ROOT
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh "" "-DBH_SORT_MATCH_TOP=2" "-DBH_SORT_MATCH_TOP=3" "-DBH_SORT_UNIFORM=1" "-DBH_SORT_UNIFORM=1 -DBH_SORT_MATCH_TOP=2"
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_sort" --clock-control none --csv --log-file gpurun_out/sort_ll_cfg3.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; python tools/sort_ll.py gpurun_out/sort_ll_cfg3.csv
