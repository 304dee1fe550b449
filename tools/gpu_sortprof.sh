cd $GRAFT_REPO_ROOT
python tools/step_cfg.py cfg3 1 > gpurun_out/sp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"k_sort|k_scan" --clock-control none --csv --log-file gpurun_out/sort_launches_cfg3.csv python tools/step_cfg.py cfg3 1 > gpurun_out/sp_ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sort_pass -s 9 -c 2 -o gpurun_out/sortpass python tools/step_cfg.py cfg3 1 > gpurun_out/sp_ncu2.log 2>&1
echo done
