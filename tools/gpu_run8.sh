cd $GRAFT_REPO_ROOT
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_sort|k_scan" --clock-control none --csv --log-file gpurun_out/sl3_hist2.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
python tools/sort_ll.py gpurun_out/sl3_hist2.csv > gpurun_out/sl3_hist2.txt; cat gpurun_out/sl3_hist2.txt
AB_CONFIGS="cfg2 cfg3" bash tools/walk_ab.sh "-DBH_W9_PC30=0" "" "-DBH_W9_BULK=1"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo done
