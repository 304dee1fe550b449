cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_sort.py -x -q 2>&1 | tail -2
for v in "3 0" "3 1" "2 1"; do set -- $v
BH_SORT_MINB=$1 BH_SORT_MATCH=$2 python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && \
BH_SORT_MINB=$1 BH_SORT_MATCH=$2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_sort" --clock-control none --csv --log-file gpurun_out/sl3_$1_$2.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1
python tools/sort_ll.py gpurun_out/sl3_$1_$2.csv | tail -4
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo done
