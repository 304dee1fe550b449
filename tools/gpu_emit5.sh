cd $GRAFT_REPO_ROOT
for f in "" "-DBH_EMIT_THREADS=512" "-DBH_EMIT_THREADS=1024"; do
BH_NVCC_EXTRA="$f" python -m paper_2203_08966_b200.build_lib > /dev/null 2>&1 || echo BUILD FAILED
python tools/step_cfg.py cfg3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_emit_mark|k_mom_lists" --csv --log-file gpurun_out/e_ll.csv python tools/step_cfg.py cfg3 1 > /dev/null 2>&1; echo "[$f]"; grep -E "k_" gpurun_out/e_ll.csv | awk -F'","' '{print substr($5,1,30), $(NF)}' | tail -2
done
