cd $GRAFT_REPO_ROOT
for f in "" "-DBH_HIL_MINB=2"; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hilbert|k_walk9" --csv --log-file gpurun_out/hil_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; echo "[$f]"; grep -E "k_hilbert|k_walk9" gpurun_out/hil_ll.csv | awk -F'","' '{print substr($5,1,30), $(NF)}' | tail -2
done
