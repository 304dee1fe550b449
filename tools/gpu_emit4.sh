cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_walk_only.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "walk_only or fp32 or scale or leaf or bucket or cfg or overflow" 2>&1 | tail -2
AB_CONFIGS="cfg3 cfg4" bash tools/sort_ab.sh ""
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_emit|k_bucket|k_moments|k_mom_lists|k_compact|k_nchild|k_scan_list|k_base_list|k_lcp|k_scan|k_hilbert" --csv --log-file gpurun_out/b_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; grep -E "k_" gpurun_out/b_ll.csv | awk -F'","' '{print substr($5,1,40), $(NF)}' | tail -24
