cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q 2>&1 | tail -3
for m in 3 2; do
BH_SORT_MINB=$m python tools/step_cfg.py cfg3 1 > gpurun_out/sp_plain$m.log 2>&1 && \
BH_SORT_MINB=$m ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_sort|k_scan" --clock-control none --csv --log-file gpurun_out/sort_launches_cfg3_m$m.csv python tools/step_cfg.py cfg3 1 > gpurun_out/sp_ncu1.log 2>&1
done
python tools/step_cfg.py cfg2 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_sort|k_scan" --clock-control none --csv --log-file gpurun_out/sort_launches_cfg2.csv python tools/step_cfg.py cfg2 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sort_pass -s 9 -c 1 -o gpurun_out/sortpass2 python tools/step_cfg.py cfg3 1 > gpurun_out/sp_ncu2.log 2>&1
echo done
