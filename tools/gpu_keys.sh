cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "key or order or sort or golden" 2>&1 | tail -2
for f in "-DBH_KEYS2=0" ""; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_keys" --csv --log-file gpurun_out/k_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; echo "[$f]"; grep -E "k_keys" gpurun_out/k_ll.csv | awk -F'","' '{print substr($5,1,30), $(NF)}' | tail -2
done
