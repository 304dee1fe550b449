cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg4 cfg2" bash tools/sort_ab.sh ""
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_lcp|k_emit|k_mom|k_bucket|k_compact|k_nchild|k_base|k_scan" --csv --log-file gpurun_out/b_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; grep -E "k_" gpurun_out/b_ll.csv | awk -F'","' '{print substr($5,1,40), $(NF)}' | tail -16
